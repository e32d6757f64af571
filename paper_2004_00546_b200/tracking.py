"""Host driver of the reference's hybrid loop with its own objective on the GPU
(`hybrid.py:185-290`, `optimization.py:84-112,172-189`).

`HybridTrackingEngine` owns one ``px_hybrid_*`` handle (include/paraexp.h): the serial Burgers
direct sweep with the forcing field f(x)·θ(t) and the tracking cost, every slice's adjoint
solve overlapped with the sweep (per-slice progress flags), the host planning of the frozen
J(ū_p)ᵀ actions between the sweeps (`expaction.plan_family` on the FOV box the device
returns), and the frozen-operator carry with the θ-weighted series for ∂L/∂f.

`solve_hybrid_tracking` is the solver-level entry (the reference's `solve_hybrid` with an
adjoint source, `hybrid.py:240-290`, plus the loop's cost and gradient); the loop-level entry
is `direct_adjoint_loop(..., algorithm="hybrid", objective="tracking")` (optimization.py).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .engine import current_stream_handle
from .errors import ConfigError
from .expaction import ChebyshevConfig, plan_family
from .hybrid import HybridPlan, TimeLaw, aligned_partition, slice_offsets
from .partition import RK4Config, TimePartition, partition_equidistant
from .problems import frozen_region_from_bounds
from .systems import System


@dataclass
class HybridTrackingResult:
    J: np.ndarray                   # (B,) (1/T)∫‖u − u_t‖² dt
    grad: np.ndarray                # (B, n) ∂L/∂f = (1/T)∫θ(t)·q†(t) dt
    final_state: np.ndarray         # (B, n) u(T)
    qdag0: np.ndarray               # (B, n) q†(0)
    partition: TimePartition        # the node-aligned partition the sweeps used
    offsets: np.ndarray             # (P+1,) node offsets
    timing: dict = field(default_factory=dict)
    plans: list = field(default_factory=list, repr=False)


class HybridTrackingEngine:
    """One px_hybrid handle: fixed grid, batch, slices (node offsets) and time law."""

    def __init__(self, system: System, offsets, law: TimeLaw, batch: int = 1, target_batched: bool = False):
        if system.is_linear:
            raise ConfigError("the hybrid tracking path is the Burgers testbed's (hybrid.py serial direct sweep)")
        self.lib = N.load()
        self.system = system
        self.offsets = np.ascontiguousarray(offsets, dtype=np.int32)
        self.P = len(self.offsets) - 1
        self.S = int(self.offsets[-1])
        self.B = int(batch)
        self.law = law
        self.target_batched = bool(target_batched)
        n = system.n
        self.n = n
        self.step = system.spec.T / self.S
        d = N.HybridDesc()
        d.nx = system.grid.nx
        d.ny = system.grid.ny if system.is_burgers2d else 0  # ny > 1: the two-field 2D testbed (hybrid2d.cu)
        d.hy = system.grid.hy
        d.D = system.spec.D
        d.hx = system.grid.hx
        d.T = system.spec.T
        d.batch = self.B
        d.nslices = self.P
        d.offsets = self.offsets.ctypes.data_as(ctypes.POINTER(ctypes.c_int))
        for k, v in enumerate(law.as_tuple()):
            d.law[k] = v
        d.target_batched = 1 if target_batched else 0
        try:
            import torch
            if torch.cuda.is_available():
                torch.cuda.set_device(torch.cuda.current_device())
        except ImportError:
            pass
        h = ctypes.c_void_p()
        N.check(self.lib, self.lib.px_hybrid_create(ctypes.byref(d), ctypes.byref(h)), None, hybrid=True)
        self.h = h

    def _chk(self, rc):
        N.check(self.lib, rc, self.h, hybrid=True)

    def close(self) -> None:
        if getattr(self, "h", None):
            self.lib.px_hybrid_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def get(self, fld: int, shape, stream: int | None = None) -> np.ndarray:
        out = np.empty(int(np.prod(shape)), dtype=np.float64)
        s = current_stream_handle() if stream is None else stream
        self._chk(self.lib.px_hybrid_get(self.h, fld, out.ctypes.data_as(ctypes.c_void_p), out.size,
                                         N.PX_MEM_HOST, ctypes.c_void_p(s)))
        return out.reshape(shape)

    def timing(self) -> dict:
        ms = (ctypes.c_double * 5)()
        self._chk(self.lib.px_hybrid_get_timing(self.h, ms))
        return {"direct_ms": ms[0], "slices_ms": ms[1], "total_ms": ms[2], "tail_ms": ms[3],
                "overlapped": bool(ms[4])}

    def set_inputs(self, u0, f, target, qdag_T=None, stream: int | None = None) -> None:
        """Host arrays, or a CUDA torch tensor ``target`` (then every input goes device to
        device: the (S+1)·n target is the large one)."""
        B, n = self.B, self.n
        if getattr(target, "is_cuda", False):
            return self._set_inputs_device(u0, f, target, qdag_T, stream)
        u0 = np.ascontiguousarray(np.broadcast_to(np.asarray(u0, dtype=np.float64).reshape(-1, n), (B, n)))
        f = np.ascontiguousarray(np.broadcast_to(np.asarray(f, dtype=np.float64).reshape(-1, n), (B, n)))
        tshape = (self.S + 1, B, n) if self.target_batched else (self.S + 1, n)
        target = np.ascontiguousarray(np.asarray(target, dtype=np.float64).reshape(tshape))
        q = None
        if qdag_T is not None:
            q = np.ascontiguousarray(np.broadcast_to(np.asarray(qdag_T, dtype=np.float64).reshape(-1, n), (B, n)))
        self._keep = (u0, f, target, q)  # host buffers live until the async copies complete
        s = current_stream_handle() if stream is None else stream
        self._chk(self.lib.px_hybrid_set_inputs(
            self.h, u0.ctypes.data_as(ctypes.c_void_p), f.ctypes.data_as(ctypes.c_void_p),
            target.ctypes.data_as(ctypes.c_void_p), q.ctypes.data_as(ctypes.c_void_p) if q is not None else None,
            N.PX_MEM_HOST, ctypes.c_void_p(s)))

    def _set_inputs_device(self, u0, f, target, qdag_T, stream) -> None:
        import torch
        B, n = self.B, self.n
        dev = target.device
        as_dev = lambda a: torch.as_tensor(np.ascontiguousarray(np.broadcast_to(
            np.asarray(a, dtype=np.float64).reshape(-1, n), (B, n))), device=dev)
        tshape = (self.S + 1, B, n) if self.target_batched else (self.S + 1, n)
        tg = target.to(torch.float64).reshape(tshape).contiguous()
        u, ff = as_dev(u0), as_dev(f)
        q = as_dev(qdag_T) if qdag_T is not None else None
        self._keep = (u, ff, tg, q)
        s = current_stream_handle() if stream is None else stream
        ptr = lambda t: ctypes.c_void_p(t.data_ptr()) if t is not None else None
        self._chk(self.lib.px_hybrid_set_inputs(self.h, ptr(u), ptr(ff), ptr(tg), ptr(q), N.PX_MEM_DEVICE,
                                                ctypes.c_void_p(s)))

    def direct(self, overlap: bool = True, stream: int | None = None) -> None:
        s = current_stream_handle() if stream is None else stream
        self._chk(self.lib.px_hybrid_direct(self.h, 1 if overlap else 0, ctypes.c_void_p(s)))

    def bounds(self, stream: int | None = None) -> tuple[float, float, float]:
        out = (ctypes.c_double * 3)()
        s = current_stream_handle() if stream is None else stream
        self._chk(self.lib.px_hybrid_bounds(self.h, out, ctypes.c_void_p(s)))
        return float(out[0]), float(out[1]), float(out[2])

    def plan(self, expaction: ChebyshevConfig, bounds, with_top: bool) -> list:
        """Per-slice plans of the frozen actions on the FOV box (one region for all slices)."""
        region = frozen_region_from_bounds(*bounds)
        spans = [float(self.offsets[p + 1] - self.offsets[p]) * self.step for p in range(self.P)]
        plans = plan_family(region, spans, expaction, omega=self.law.omega)
        top = self.P - 1 if with_top else self.P - 2
        for p in range(top + 1):
            pl = plans[p]
            c = N.ChebPlanC()
            c.span = pl.span
            c.substeps = pl.substeps
            c.degree = pl.degree
            c.center = pl.center
            c.scale = pl.scale
            c.sigma = pl.sigma
            be, ka = N.dptr(pl.coef_exp)
            bp, kb = N.dptr(pl.coef_phi)
            c.coef_exp, c.coef_phi = be, bp
            gc = gs = None
            keep = []
            if self.law.omega != 0.0:
                gc, kc = N.dptr(pl.coef_gc)
                gs, kd = N.dptr(pl.coef_gs)
                keep = [kc, kd]
            self._chk(self.lib.px_hybrid_set_slice_plan(self.h, p, ctypes.byref(c), gc, gs))
            del ka, kb, keep
        return plans

    def adjoint(self, stream: int | None = None) -> None:
        s = current_stream_handle() if stream is None else stream
        self._chk(self.lib.px_hybrid_adjoint(self.h, ctypes.c_void_p(s)))

    # ---- Algorithm 2 on the 2D two-field testbed (px_hybrid_nl_*) ------------------------------
    @staticmethod
    def _plan_c(pl):
        c = N.ChebPlanC()
        c.span, c.substeps, c.degree, c.center, c.scale, c.sigma = (pl.span, pl.substeps, pl.degree, pl.center,
                                                                     pl.scale, pl.sigma)
        be, ka = N.dptr(pl.coef_exp)
        bp, kb = N.dptr(pl.coef_phi)
        c.coef_exp, c.coef_phi = be, bp
        return c, (ka, kb)

    def iterate_direct(self, expaction: ChebyshevConfig, eps: float, max_iter: int = 25, min_iter: int = 2,
                       stream: int | None = None) -> list:
        """`solve_direct_nonlinear` (`nonlinear.py:69-194`): sweeps until the largest per-slice relative
        change is below ``eps`` (at least ``min_iter`` sweeps); the iterate becomes the direct trajectory.
        Returns the error history; raises `IterationDivergence` after ``max_iter`` sweeps."""
        from .errors import IterationDivergence
        from .expaction import plan_chebyshev
        s = current_stream_handle() if stream is None else stream
        self._chk(self.lib.px_hybrid_nl_init(self.h, ctypes.c_void_p(s)))
        delta = float(self.offsets[1]) * self.step
        history = []
        for it in range(1, max_iter + 1):
            region = frozen_region_from_bounds(*self.bounds(s))
            cs, k1 = self._plan_c(plan_chebyshev(region, delta, expaction))
            ch, k2 = self._plan_c(plan_chebyshev(region, self.step, expaction))
            self._chk(self.lib.px_hybrid_nl_set_plans(self.h, ctypes.byref(cs), ctypes.byref(ch)))
            del k1, k2
            err = ctypes.c_double()
            self._chk(self.lib.px_hybrid_nl_sweep(self.h, ctypes.byref(err), ctypes.c_void_p(s)))
            history.append(float(err.value))
            if err.value < eps and it >= min_iter:
                self._chk(self.lib.px_hybrid_nl_finish(self.h, ctypes.c_void_p(s)))
                return history
        raise IterationDivergence(history)

    def run_nonlinear(self, u0, f, target, expaction: ChebyshevConfig, eps: float, max_iter: int = 25,
                      min_iter: int = 2) -> dict:
        self.set_inputs(u0, f, target, None)
        history = self.iterate_direct(expaction, eps, max_iter, min_iter)
        b = self.bounds()
        plans = self.plan(expaction, b, False) if self.P > 1 else []
        self.adjoint()
        B, n = self.B, self.n
        return {"J": self.get(N.PX_HFIELD_J, (B,)), "grad": self.get(N.PX_HFIELD_GRAD, (B, n)),
                "uT": self.get(N.PX_HFIELD_UT, (B, n)), "qdag0": self.get(N.PX_HFIELD_QDAG0, (B, n)),
                "timing": self.timing(), "plans": plans, "bounds": b, "history": history}

    def run(self, u0, f, target, expaction: ChebyshevConfig, qdag_T=None, overlap: bool = True) -> dict:
        self.set_inputs(u0, f, target, qdag_T)
        self.direct(overlap)
        b = self.bounds()
        plans = self.plan(expaction, b, qdag_T is not None) if (self.P > 1 or qdag_T is not None) else []
        self.adjoint()
        B, n = self.B, self.n
        return {"J": self.get(N.PX_HFIELD_J, (B,)), "grad": self.get(N.PX_HFIELD_GRAD, (B, n)),
                "uT": self.get(N.PX_HFIELD_UT, (B, n)), "qdag0": self.get(N.PX_HFIELD_QDAG0, (B, n)),
                "timing": self.timing(), "plans": plans, "bounds": b}


_TRACKING: dict = {}


def get_tracking_engine(system: System, offsets, law: TimeLaw, batch: int, target_batched: bool):
    key = (system.grid, system.spec, tuple(int(o) for o in offsets), law, batch, target_batched)
    eng = _TRACKING.get(key)
    if eng is None:
        eng = HybridTrackingEngine(system, offsets, law, batch, target_batched)
        _TRACKING[key] = eng
    return eng


def release_tracking_engines() -> None:
    for e in _TRACKING.values():
        e.close()
    _TRACKING.clear()


def _offsets_for(system: System, plan: HybridPlan | None, N: int, rk: RK4Config):
    part = plan.partition if plan is not None else partition_equidistant(system.spec.T, N)
    offs = slice_offsets(part, rk.dt)
    return offs, aligned_partition(offs, system.spec.T, plan.k if plan is not None else None)


def solve_hybrid_tracking(system: System, u0, f, target, plan: HybridPlan | None = None, N: int = 1,
                          rk: RK4Config | None = None, expaction: ChebyshevConfig | None = None,
                          law: TimeLaw | None = None, qdag_T=None, overlap: bool = True) -> HybridTrackingResult:
    """The reference's hybrid solve with its tracking objective on the GPU (`hybrid.py:240-290`
    with adj_source = 2(q − q_true), `optimization.py:172-189`).

    ``f``: forcing field(s) (n,) or (B, n); ``target``: the tracking target on the serial sweep's
    nodes, (S+1, n) shared or (S+1, B, n); ``plan``: a `HybridPlan` (geometric partition) or
    None for ``N`` equal slices; ``law``: the forcing's time law (default constant);
    ``qdag_T``: optional adjoint terminal data (the final span, `hybrid.py:232-233`)."""
    if rk is None:
        raise ConfigError("rk: an RK4Config(dt) is required (fixed-step RK4)")
    law = law or TimeLaw.constant()
    expaction = expaction or ChebyshevConfig(tol=1e-12)
    if not isinstance(expaction, ChebyshevConfig):
        raise ConfigError("expaction: the frozen J(ū_p)ᵀ actions are Chebyshev series")
    f = np.atleast_2d(np.asarray(f, dtype=np.float64))
    if f.shape[-1] != system.n:
        raise ValueError("f must be a forcing field of n points (or B fields)")
    B = f.shape[0]
    offs, part = _offsets_for(system, plan, N, rk)
    S = int(offs[-1])
    if not getattr(target, "is_cuda", False):
        target = np.asarray(target, dtype=np.float64)
    if tuple(target.shape) == (S + 1, system.n):
        batched = False
    elif tuple(target.shape) == (S + 1, B, system.n):
        batched = True
    else:
        raise ValueError(f"target must be given on the {S + 1} nodes of the sweep: (S+1, n) or (S+1, B, n)")
    eng = get_tracking_engine(system, offs, law, B, batched)
    r = eng.run(u0, f, target, expaction, qdag_T, overlap)
    return HybridTrackingResult(J=r["J"], grad=r["grad"], final_state=r["uT"], qdag0=r["qdag0"], partition=part,
                                offsets=offs, timing=r["timing"], plans=r["plans"])


def solve_nonlinear_tracking(system: System, u0, f, target, N: int = 1, rk: RK4Config | None = None,
                             expaction: ChebyshevConfig | None = None, law: TimeLaw | None = None,
                             eps: float = 1e-3, max_iter: int = 25, min_iter: int = 2) -> HybridTrackingResult:
    """The reference's loop with algorithm "nonlinear" on its 2D two-field Burgers testbed
    (`optimization.py:206-231`): the iterative nonlinear direct (Algorithm 2, `nonlinear.py:69-194`)
    on ``N`` equal slices, then `solve_adjoint_varying` with the source 2(q − q_t) and zero terminal
    data (the hybrid's adjoint form), the tracking cost and ∂L/∂f. ``timing["history"]`` holds the
    sweeps' errors. Whole RK4 steps per slice (on chip for nx·ny ≤ 2048, per-stage launches above)."""
    if rk is None:
        raise ConfigError("rk: an RK4Config(dt) is required (fixed-step RK4)")
    if not getattr(system, "is_burgers2d", False):
        raise ConfigError("solve_nonlinear_tracking: the two-field 2D Burgers testbed (1D: algorithm='nonlinear' "
                          "with the terminal objective)")
    if eps <= 0:
        raise ValueError("eps must be positive")
    law = law or TimeLaw.constant()
    expaction = expaction or ChebyshevConfig(tol=1e-12)
    f = np.atleast_2d(np.asarray(f, dtype=np.float64))
    if f.shape[-1] != system.n:
        raise ValueError("f must be a forcing field of n points (or B fields)")
    B = f.shape[0]
    steps = max(1, int(np.ceil(system.spec.T / (N * rk.dt) - 1e-9)))
    offs = (np.arange(N + 1) * steps).astype(np.int32)
    S = int(offs[-1])
    if abs(system.spec.T / S - rk.dt) > 1e-12 * rk.dt:
        raise ConfigError(f"rk.dt must divide the slice width T/N into whole steps (nearest: {system.spec.T / S!r})")
    target = np.asarray(target, dtype=np.float64)
    if tuple(target.shape) == (S + 1, system.n):
        batched = False
    elif tuple(target.shape) == (S + 1, B, system.n):
        batched = True
    else:
        raise ValueError(f"target must be given on the {S + 1} nodes of the sweep: (S+1, n) or (S+1, B, n)")
    eng = get_tracking_engine(system, offs, law, B, batched)
    r = eng.run_nonlinear(u0, f, target, expaction, eps, max_iter, min_iter)
    timing = dict(r["timing"], history=r["history"])
    return HybridTrackingResult(J=r["J"], grad=r["grad"], final_state=r["uT"], qdag0=r["qdag0"],
                                partition=partition_equidistant(system.spec.T, N), offsets=offs, timing=timing,
                                plans=r["plans"])


def synthesize_trajectory(system: System, f_true, rk: RK4Config, law: TimeLaw | None = None, u0=None) -> np.ndarray:
    """The tracking target: the serial sweep's node trajectory (S+1, B, n) of the system under
    ``f_true``·θ(t) (`optimization.py:66-80`, on the GPU). The linear testbed records it with the
    one-slice tracking loop (``f_true``: K values per member; a field system takes the field)."""
    law = law or TimeLaw.constant()
    f = np.atleast_2d(np.asarray(f_true, dtype=np.float64))
    B, n = f.shape[0], system.n
    if system.is_linear:
        from .optimization import SERIAL, direct_adjoint_loop
        from .partition import slice_steps
        S = slice_steps(system.spec.T, rk.dt)
        r = direct_adjoint_loop(system, f, np.zeros((S + 1, n)), SERIAL, rk=rk, u0=u0, objective="tracking",
                                time_law=law)
        return r.stats["trajectory"].numpy()
    offs, _ = _offsets_for(system, None, 1, rk)
    S = int(offs[-1])
    u0 = np.zeros(n) if u0 is None else u0
    eng = get_tracking_engine(system, offs, law, B, False)
    eng.set_inputs(u0, f, np.zeros((S + 1, n)))
    eng.direct(overlap=False)
    return eng.get(N.PX_HFIELD_TRAJ, (S + 1, B, n))


def pilot_times(system: System, steps: int, rk: RK4Config, repeats: int, law: TimeLaw) -> tuple[float, float]:
    """Device seconds per unit of simulated time of the serial direct sweep and of one slice's
    adjoint solve, on a pilot span of ``steps`` steps (for `hybrid.estimate_k`)."""
    import math
    from dataclasses import replace

    spec = replace(system.spec, T=steps * rk.dt)
    sysp = System(system.grid, spec, system.basis)
    offs = np.array([0, steps], dtype=np.int32)
    eng = HybridTrackingEngine(sysp, offs, law, 1, False)
    try:
        if system.is_burgers2d:
            X, Y = system.grid.coordinates()
            u0 = np.concatenate([0.5 * np.sin(X), 0.5 * np.sin(Y)])
        else:
            u0 = 0.5 * np.sin(system.grid.x1())
        f = np.zeros(system.n)
        tgt = np.zeros((steps + 1, system.n))
        dirs, adjs = [], []
        for _ in range(max(1, repeats) + 1):   # the first run warms up
            eng.set_inputs(u0, f, tgt)
            eng.direct(overlap=False)
            t = eng.timing()
            dirs.append(t["direct_ms"])
            adjs.append(t["slices_ms"])
        span = steps * rk.dt
        t_dir = float(np.median(dirs[1:])) / 1e3 / span
        t_adj = float(np.median(adjs[1:])) / 1e3 / span
        if not (math.isfinite(t_dir) and t_dir > 0):
            from .errors import PilotTooShort
            raise PilotTooShort("pilot direct sweep could not be timed; widen pilot_fraction")
        return t_dir, t_adj
    finally:
        eng.close()
