"""GPU engine: one native handle per (problem, rank), driven phase by phase.

Replaces the reference's worker transport for this path (`workers.py:298-346`,
Python threads or forked processes exchanging n-vectors): the P time slices of a
rank run as one batched kernel grid on its GPU, the neighbour chains become one
summed-chain carry per sweep, and the only inter-rank exchange is an allreduce
of the u(T) partials (direct) and of the q†(0)/∫q†/gradient partials (adjoint),
done here with ``torch.distributed`` (NCCL over NVLink) on the handle's device
buffers when ``world > 1``.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .errors import CollectiveFailure, ConfigError, IntegrationFailure, IterationDivergence, NativeUnavailable
from .expaction import ChebPlan, ChebyshevConfig, KrylovConfig, KrylovPlan, plan_chebyshev, plan_for
from .partition import balanced_blocks, partition_equidistant, rank_block, slice_steps
from .problems import ADVECTION_DIFFUSION, frozen_region_from_bounds
from .systems import System


def _torch():
    try:
        import torch
        return torch
    except Exception:  # pragma: no cover - torch is in the image
        return None


def current_stream_handle() -> int:
    """The caller's current CUDA stream (torch's), or 0 (legacy default stream)."""
    torch = _torch()
    if torch is not None and torch.cuda.is_available():
        return int(torch.cuda.current_stream().cuda_stream)
    return 0


def check_rk4_stability(region, h: float) -> None:
    """Raise ConfigError if the classical RK4 step h is unstable on the spectral
    enclosure: max |R(hλ)| over its boundary > 1 (R(z) = 1 + z + z²/2 + z³/6 + z⁴/24)."""
    z = h * region.boundary(2048)
    R = 1 + z * (1 + z * (0.5 + z * (1.0 / 6.0 + z / 24.0)))
    amp = float(np.max(np.abs(R)))
    if amp > 1.0 + 1e-9:
        raise ConfigError(f"RK4 step h={h:.3g} is unstable on this operator (max |R(hλ)| = {amp:.4g}); "
                          "decrease dt")


class _DeviceView:
    """__cuda_array_interface__ over a native device buffer (for torch/NCCL)."""

    def __init__(self, ptr: int, count: int):
        self.__cuda_array_interface__ = {
            "shape": (count,), "typestr": "<f8", "data": (ptr, False), "version": 3, "strides": None,
        }


@dataclass(frozen=True)
class EngineSpec:
    system: System
    P: int
    dt: float
    expaction: ChebyshevConfig | KrylovConfig
    batch: int = 1
    rank: int = 0
    world: int = 1
    boundary_states: bool = False
    direct: str = "serial"      # Burgers: "serial" sweep or "iterative" (Algorithm 2)
    nl_eps: float = 1e-3
    nl_max_iter: int = 25
    nl_min_iter: int = 2
    local_blocks: int = 0       # 0: automatic (concurrent block carries for Krylov); 1: sequential scan
    variants: tuple = ()        # ((name, value), …) kernel variants (_native.VARIANTS), e.g. (("march2", 2),)
    z_accum: bool = False       # 2D adjoint ∫ by a per-lane accumulator instead of the closed form
    law: tuple = (1.0, 0.0, 0.0, 0.0)  # forcing time law θ(t) = α + β sin ωt + γ cos ωt (linear testbed)

    @property
    def has_law(self) -> bool:
        return tuple(self.law[:3]) != (1.0, 0.0, 0.0)

    @property
    def nsteps(self) -> int:
        return slice_steps(self.system.spec.T / self.P, self.dt)


# developer overrides of the kernel variants (tools/ experiments); tests use EngineSpec.variants
ENV_VARIANTS = {"PX_MARCH2": "march2", "PX_M2_COLS": "march_cols", "PX_M2_BAND": "march_band",
                "PX_CM_TERMS": "cheb_terms", "PX_CM_TERMS_PHI": "cheb_terms_phi", "PX_CM_STRIP": "cheb_strip", "PX_CM_BAND": "cheb_band",
                "PX_SCAN1D_CLUSTER": "scan1d_cluster", "PX_BURGERS_CLUSTER": "burgers_cluster",
                "PX_KRYLOV_ORTHO": "krylov_ortho"}


def allreduce_sum(tensors, group=None, stream=None) -> None:
    """In-place SUM allreduce of each tensor over the process group (NCCL on GPU), ordered
    after the work enqueued on ``stream`` (the native kernels' stream) when one is given."""
    import torch
    import torch.distributed as dist
    ctx = None
    if stream and torch.cuda.is_available() and any(t.is_cuda for t in tensors):
        ctx = torch.cuda.stream(torch.cuda.ExternalStream(stream))
    if ctx is None:
        for t in tensors:
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
        return
    with ctx:
        for t in tensors:
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)


def agree_status(code: int, group=None) -> int:
    """Every rank contributes ``code`` (its failure code, or a large sentinel when healthy);
    returns the MIN over ranks, the same value on every rank. On a CUDA (NCCL) group the
    flag travels in a device tensor."""
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    t = torch.tensor([code], dtype=torch.int64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
    return int(t.item())


_HEALTHY = 1 << 62


def distributed_gradient(eng, stream=None, group=None, want_fields: bool = True, reduce=allreduce_sum,
                         agree=agree_status) -> None:
    """One sharded gradient evaluation: each rank runs its slice
    block, the u(T) partials are summed, every rank finishes the direct sweep
    identically, runs its adjoint block and the adjoint partials are summed.

    ``eng`` provides ``direct_partial / finish_direct / adjoint_partial /
    finish_adjoint`` and ``view(field)`` (a tensor aliasing the field's buffer);
    the partial conventions are the C ABI's (`px_finish_*` add the q0 / q†_T terms
    once, after the reduction).

    Fail-fast on every rank (the reference aborts all workers, `workers.py:140-160`): before
    each collective the ranks agree on a status word (``agree``: MIN over ranks of
    phase·world + rank for a failed rank); if any rank failed, every rank raises
    ``CollectiveFailure(first failing rank, phase, cause)`` instead of entering the reduction
    its peer will never join.
    """
    rank = getattr(getattr(eng, "spec", None), "rank", 0)
    world = max(1, getattr(getattr(eng, "spec", None), "world", 1))
    stages = (
        (("direct", lambda: eng.direct_partial(stream)),),
        (("finish direct", lambda: eng.finish_direct(stream)), ("adjoint", lambda: eng.adjoint_partial(stream))),
        (("finish adjoint", lambda: eng.finish_adjoint(stream)),),
    )
    collectives = (
        ("direct allreduce", lambda: reduce([eng.view(f) for f in eng.direct_reduce_fields()], group, stream)),
        ("adjoint allreduce",
         lambda: reduce([eng.view(f) for f in eng.adjoint_reduce_fields(want_fields)], group, stream)),
    )
    names = [n for st in stages for n, _ in st] + [n for n, _ in collectives]
    for i, stage in enumerate(stages):
        code, cause = _HEALTHY, None
        for name, run in stage:
            try:
                run()
            except Exception as e:  # noqa: BLE001 - mapped onto the reference's CollectiveFailure
                code, cause = names.index(name) * world + rank, e
                break
        if i == len(stages) - 1:
            if cause is not None:
                raise CollectiveFailure(rank, names[code // world], cause) from cause
            return
        cname, crun = collectives[i]
        first = agree(code, group)
        if first != _HEALTHY:
            failed_rank, phase = first % world, names[first // world]
            err = cause if failed_rank == rank and cause is not None else RuntimeError(
                f"rank {failed_rank} failed in {phase}; aborting the collective solve")
            raise CollectiveFailure(failed_rank, phase, err) from cause
        try:
            crun()
        except Exception as e:  # noqa: BLE001
            raise CollectiveFailure(rank, cname, e) from e


class ParaexpEngine:
    """Owns one ``px_handle``; computes gradients of J = ½‖u(T) − u_target‖²."""

    def __init__(self, spec: EngineSpec):
        self.spec = spec
        self.tracking = False  # px_set_tracking_target: the reference's linear loop objective
        self.lib = N.load()
        sysm = spec.system
        grid = sysm.grid
        if spec.world > 1 and spec.world > spec.P:
            raise ConfigError(f"world={spec.world} exceeds P={spec.P} slices")
        p0, p1 = rank_block(spec.P, spec.rank, spec.world)
        self.p0, self.p1 = p0, p1
        if sysm.is_linear:
            check_rk4_stability(sysm.region(), sysm.spec.T / spec.P / spec.nsteps)
        self.n = grid.npoints
        self.B = spec.batch
        self.K = sysm.basis.K
        d = N.ProblemDesc()
        d.kind = N.PX_KIND_ADVDIFF if sysm.spec.kind == ADVECTION_DIFFUSION else N.PX_KIND_BURGERS
        d.nx, d.ny = grid.nx, grid.ny
        for i, v in enumerate(sysm.A.as_tuple()):
            d.stencil[i] = v
        d.D = sysm.spec.D
        d.hx = grid.hx
        d.T = sysm.spec.T
        d.P = spec.P
        d.nsteps = spec.nsteps
        d.p_begin, d.p_end = p0, p1
        d.batch = spec.batch
        d.K = self.K
        d.basis_rows_x = sysm.basis.tx.shape[0]
        d.basis_rows_y = sysm.basis.ty.shape[0]
        krylov = isinstance(spec.expaction, KrylovConfig)
        d.expaction = N.PX_EXP_KRYLOV if krylov else N.PX_EXP_CHEBYSHEV
        d.krylov_m = spec.expaction.m if krylov else 0
        field_ctl = getattr(sysm.basis, "is_field", False)
        d.flags = (N.PX_FLAG_BOUNDARY_STATES if spec.boundary_states else 0) | (
            N.PX_FLAG_Z_ACCUM if spec.z_accum or os.environ.get("PX_Z_ACCUM") == "1" else 0) | (
            N.PX_FLAG_FIELD_CONTROL if field_ctl else 0)
        if spec.has_law and not sysm.is_linear:
            raise ConfigError("time_law: the linear testbed's loop (Burgers: objective='tracking', hybrid)")
        if spec.has_law and isinstance(spec.expaction, KrylovConfig):
            raise ConfigError("time_law: needs Chebyshev exp-actions (their time-law integral series)")
        self._desc = d
        torch = _torch()
        if torch is not None and torch.cuda.is_available():
            # libparaexp links cudart statically: it allocates on the device whose primary
            # context is current on this thread, so make torch's device (LOCAL_RANK under
            # torchrun) current before the handle allocates
            torch.cuda.set_device(torch.cuda.current_device())
            torch.cuda.current_stream().synchronize()
        h = ctypes.c_void_p()
        N.check(self.lib, self.lib.px_create(ctypes.byref(d), ctypes.byref(h)))
        self.h = h
        for env, name in ENV_VARIANTS.items():
            if os.environ.get(env):
                self.set_variant(name, int(os.environ[env]))
        for name, value in spec.variants:
            self.set_variant(name, value)
        if not field_ctl:
            tx, _a = N.dptr(sysm.basis.tx)
            ty, _b = N.dptr(sysm.basis.ty)
            ix, _c = N.iptr(sysm.basis.ix)
            iy, _d = N.iptr(sysm.basis.iy)
            N.check(self.lib, self.lib.px_set_basis(h, tx, ty, ix, iy), h)
        if spec.has_law:
            law, _e = N.dptr(np.asarray(spec.law, dtype=np.float64))
            N.check(self.lib, self.lib.px_set_time_law(h, law), h)
        self.plans: dict[int, ChebPlan | KrylovPlan] = {}
        self._keep = []
        self._adjoint_mode = "absorbed"
        self.nl_history: list[float] = []
        if spec.direct not in ("serial", "iterative"):
            raise ConfigError(f"unknown direct solver {spec.direct!r}")
        if spec.direct == "iterative" and (sysm.is_linear or spec.world != 1):
            raise ConfigError("the iterative direct (Algorithm 2) is the one-rank Burgers path")
        if sysm.is_linear:
            region = sysm.region()
            delta = sysm.spec.T / spec.P
            if p1 - p0 > 1:  # carries between this rank's slices (none for one slice: serial)
                self._set_plan(N.PX_PLAN_SLICE, self._plan(region, delta))
            if p1 < spec.P:
                self._set_plan(N.PX_PLAN_LONG_DIRECT, self._plan(region, (spec.P - p1) * delta))
            if p0 > 0:
                self._set_plan(N.PX_PLAN_LONG_ADJOINT, self._plan(region, p0 * delta))
            lb = self._local_blocks(p1 - p0)
            self.block_sizes = [p1 - p0]
            if lb > 1:
                sizes = self._block_sizes(region, p1 - p0, lb, delta)
                for k in range(1, lb):  # slot k−1: the last k direct blocks (= the first k adjoint blocks)
                    self._set_plan(N.PX_PLAN_BLOCK_LONG + k - 1, self._plan(region, sum(sizes[lb - k:]) * delta))
                if len(set(sizes)) == 1:
                    N.check(self.lib, self.lib.px_set_local_blocks(self.h, lb), self.h)
                else:
                    arr, _keep = N.iptr(np.asarray(sizes, dtype=np.int32))
                    N.check(self.lib, self.lib.px_set_local_block_sizes(self.h, lb, arr), self.h)
                self.block_sizes = sizes
            self.local_blocks = lb

    def _local_blocks(self, Pl: int) -> int:
        """Concurrent block carries inside this GPU (`px_set_local_blocks`). Automatic: 4
        blocks for the Krylov path (its Arnoldi kernels are latency-bound and leave the GPU
        mostly idle, and a Krylov long span costs ≈ 1/8 of the slices it spans); the
        Chebyshev march already fills the GPU and stays sequential. PX_LOCAL_BLOCKS overrides."""
        spec = self.spec
        env = os.environ.get("PX_LOCAL_BLOCKS")
        want = int(env) if env else spec.local_blocks
        if want == 0:
            want = 4 if isinstance(spec.expaction, KrylovConfig) else 1
        if self.spec.system.grid.dim != 2 or spec.boundary_states:
            return 1
        return max(1, min(want, N.PX_MAX_LOCAL_BLOCKS, Pl))

    def _block_sizes(self, region, Pl: int, lb: int, delta: float) -> list[int]:
        """Local block sizes: near-equal contiguous blocks (`rank_block`) by default;
        PX_BALANCED_BLOCKS=1 balances each block's carries against its long span
        (`partition.balanced_blocks`, ρ = the long span's cost per slice spanned from the
        planner). Measured on config 4 (4 blocks): equal 153 ms, balanced 156 ms per gradient —
        the concurrent blocks share the GPU, so the total work, not one block's chain, decides."""
        if os.environ.get("PX_BALANCED_BLOCKS") != "1":
            return [b - a for a, b in (rank_block(Pl, g, lb) for g in range(lb))]
        k = max(1, Pl // lb)
        one = self._plan(region, delta)
        span = self._plan(region, k * delta)
        rho = span.terms / (k * max(one.terms, 1))
        return balanced_blocks(Pl, lb, rho)

    def set_variant(self, name: str, value: int) -> None:
        """Select a kernel variant of this handle (``_native.VARIANTS``; px_set_variant)."""
        if name not in N.VARIANTS:
            raise ValueError(f"unknown kernel variant {name!r}; known: {sorted(N.VARIANTS)}")
        N.check(self.lib, self.lib.px_set_variant(self.h, N.VARIANTS[name], int(value)), self.h)

    def variant(self, name: str) -> int:
        v = ctypes.c_int()
        N.check(self.lib, self.lib.px_get_variant(self.h, N.VARIANTS[name], ctypes.byref(v)), self.h)
        return int(v.value)

    # -- plans ---------------------------------------------------------------

    def _plan(self, region, span):
        return plan_for(region, span, self.spec.expaction, base_span=self.spec.system.spec.T / self.spec.P,
                        omega=self.spec.law[3] if self.spec.has_law else 0.0)

    def _set_plan(self, slot: int, plan) -> None:
        self.plans[slot] = plan
        if isinstance(plan, KrylovPlan):
            N.check(self.lib, self.lib.px_set_krylov_plan(self.h, slot, plan.span, plan.substeps), self.h)
            return
        be, ka = N.dptr(plan.coef_exp)
        bp, kb = N.dptr(plan.coef_phi)
        c = N.ChebPlanC(plan.span, plan.substeps, plan.degree, plan.center, plan.scale, plan.sigma, be, bp)
        N.check(self.lib, self.lib.px_set_cheb_plan(self.h, slot, ctypes.byref(c)), self.h)
        if plan.coef_gc is not None:
            gc, kc = N.dptr(plan.coef_gc)
            gs, kd = N.dptr(plan.coef_gs)
            N.check(self.lib, self.lib.px_set_cheb_plan_law(self.h, slot, gc, gs), self.h)

    # -- inputs / outputs ----------------------------------------------------

    def set_inputs(self, u0, u_target, ctrl, stream: int | None = None) -> None:
        """numpy arrays (host) or CUDA torch tensors (device)."""
        self._detach_snapshots()
        s = current_stream_handle() if stream is None else stream
        torch = _torch()
        if torch is not None and isinstance(u0, torch.Tensor) and u0.is_cuda:
            for t in (u0, u_target, ctrl):
                if t.dtype != torch.float64 or not t.is_contiguous():
                    raise ValueError("device inputs must be contiguous float64 tensors")
            if ctrl.numel() != self.B * self.K or u0.numel() != self.n or u_target.numel() != self.n:
                raise ValueError("input sizes do not match the problem")
            rc = self.lib.px_set_inputs(self.h, u0.data_ptr(), u_target.data_ptr(), ctrl.data_ptr(),
                                        N.PX_MEM_DEVICE, s)
            self._keep = [u0, u_target, ctrl]
        else:
            a = np.ascontiguousarray(u0, dtype=np.float64).ravel()
            b = np.ascontiguousarray(u_target, dtype=np.float64).ravel()
            c = np.ascontiguousarray(ctrl, dtype=np.float64).reshape(-1)
            if a.size != self.n or b.size != self.n or c.size != self.B * self.K:
                raise ValueError("input sizes do not match the problem")
            rc = self.lib.px_set_inputs(self.h, a.ctypes.data, b.ctypes.data, c.ctypes.data,
                                        N.PX_MEM_HOST, s)
            self._keep = [a, b, c]
        N.check(self.lib, rc, self.h)

    def set_tracking_target(self, target, stream: int | None = None) -> None:
        """The tracking objective (`px_set_tracking_target`, the reference's linear loop): the
        target trajectory on the RK4 nodes, (S+1, n) shared or (S+1, B, n) per member, numpy or a
        contiguous float64 CUDA tensor; None restores the terminal objective."""
        self._detach_snapshots()
        s = current_stream_handle() if stream is None else stream
        if target is None:
            N.check(self.lib, self.lib.px_set_tracking_target(self.h, None, 0, N.PX_MEM_HOST, s), self.h)
            self.tracking = False
            return
        S = self.spec.P * self.spec.nsteps
        torch = _torch()
        dev = torch is not None and isinstance(target, torch.Tensor) and target.is_cuda
        if dev:
            if target.dtype != torch.float64 or not target.is_contiguous():
                raise ValueError("a device target must be a contiguous float64 tensor")
            t, cnt, mem = target, target.numel(), N.PX_MEM_DEVICE
        else:
            t = np.ascontiguousarray(target, dtype=np.float64)
            cnt, mem = t.size, N.PX_MEM_HOST
        if cnt == (S + 1) * self.n:
            per = 0
        elif cnt == (S + 1) * self.B * self.n:
            per = 1
        else:
            raise ValueError(f"tracking target: (S+1, n) or (S+1, B, n) values with S = {S}")
        ptr = t.data_ptr() if dev else t.ctypes.data
        N.check(self.lib, self.lib.px_set_tracking_target(self.h, ptr, per, mem, s), self.h)
        self._keep.append(t)
        self.tracking = True

    def field_count(self, field: int) -> int:
        p = ctypes.c_void_p()
        cnt = ctypes.c_size_t()
        N.check(self.lib, self.lib.px_buffer(self.h, field, ctypes.byref(p), ctypes.byref(cnt)), self.h)
        return int(cnt.value)

    def view(self, field: int):
        return self.device_view(field)

    def device_view(self, field: int):
        """Torch CUDA tensor aliasing a native device buffer (no copy)."""
        torch = _torch()
        p = ctypes.c_void_p()
        cnt = ctypes.c_size_t()
        N.check(self.lib, self.lib.px_buffer(self.h, field, ctypes.byref(p), ctypes.byref(cnt)), self.h)
        return torch.as_tensor(_DeviceView(int(p.value), int(cnt.value)), device="cuda")

    def get(self, field: int, stream: int | None = None) -> np.ndarray:
        s = current_stream_handle() if stream is None else stream
        cnt = self.field_count(field)
        out = np.empty(cnt, dtype=np.float64)
        N.check(self.lib, self.lib.px_get(self.h, field, out.ctypes.data, cnt, N.PX_MEM_HOST, s), self.h,
                t=self.spec.system.spec.T)
        return out

    def stats(self) -> dict:
        st = N.Stats()
        N.check(self.lib, self.lib.px_get_stats(self.h, ctypes.byref(st)), self.h)
        return st.as_dict()

    def set_graphs(self, enable: bool) -> None:
        """CUDA-graph replay of the single-rank gradient (default on)."""
        N.check(self.lib, self.lib.px_set_graphs(self.h, 1 if enable else 0), self.h)

    def set_timing(self, enable, kernels: bool = False) -> None:
        """Phase timing (CUDA events around each sweep phase); ``kernels`` adds events around
        every launch of the fused RK4 march and the Chebyshev passes (eager, no graph)."""
        mode = (2 if kernels else 1) if enable else 0
        N.check(self.lib, self.lib.px_set_timing(self.h, mode), self.h)

    def kernel_timing(self, kclass: int) -> tuple[float, int]:
        """(device ms, launches) of one kernel class since the last call (timing with kernels)."""
        ms = ctypes.c_double()
        cnt = ctypes.c_uint64()
        N.check(self.lib, self.lib.px_get_kernel_timing(self.h, kclass, ctypes.byref(ms), ctypes.byref(cnt)), self.h)
        return float(ms.value), int(cnt.value)

    def timing(self) -> dict:
        """Per-phase device time (CUDA events around each sweep phase) since the last call."""
        t = N.Timing()
        N.check(self.lib, self.lib.px_get_timing(self.h, ctypes.byref(t)), self.h)
        return t.as_dict()

    def reset_stats(self) -> None:
        N.check(self.lib, self.lib.px_reset_stats(self.h), self.h)

    # -- phases --------------------------------------------------------------

    # Phase-level entry points (a rank's partial, then the finish after the caller's
    # reduction). ``distributed_gradient`` chains them with an NCCL allreduce.

    def direct_partial(self, stream: int | None = None) -> None:
        self._detach_snapshots()
        s = current_stream_handle() if stream is None else stream
        if self.spec.direct == "iterative":
            self.direct_iterative(s)
            return
        N.check(self.lib, self.lib.px_direct(self.h, s), self.h)

    def direct_iterative(self, stream: int | None = None) -> list[float]:
        """Algorithm 2 (`nonlinear.py:149-194`): Jacobian-augmented sweeps until the
        max-over-slices relative change < eps (and ≥ min_iter sweeps); the J(ū_p)
        actions are planned on the host from each iterate's slice means."""
        self._detach_snapshots()
        s = current_stream_handle() if stream is None else stream
        spec = self.spec
        cfg = spec.expaction
        if not isinstance(cfg, ChebyshevConfig):
            raise ConfigError("the iterative direct uses the Chebyshev action")
        delta = spec.system.spec.T / spec.P
        hstep = delta / spec.nsteps
        N.check(self.lib, self.lib.px_nl_init(self.h, s), self.h)
        history: list[float] = []
        err = ctypes.c_double()
        for it in range(1, spec.nl_max_iter + 1):
            N.check(self.lib, self.lib.px_nl_prepare(self.h, s), self.h)
            lo, hi, im = self.get(N.PX_FIELD_FROZEN_BOUNDS, s)
            if not np.all(np.isfinite([lo, hi, im])):
                raise IntegrationFailure(spec.system.spec.T, "non-finite iterate")
            region = frozen_region_from_bounds(float(lo), float(hi), float(im))
            self._set_plan(N.PX_PLAN_NL_SLICE, plan_chebyshev(region, delta, cfg))
            self._set_plan(N.PX_PLAN_NL_STEP, plan_chebyshev(region, hstep, cfg))
            N.check(self.lib, self.lib.px_nl_sweep(self.h, ctypes.byref(err), s), self.h, t=spec.system.spec.T)
            history.append(float(err.value))
            if err.value < spec.nl_eps and it >= spec.nl_min_iter:
                break
        else:
            self.nl_history = history
            raise IterationDivergence(history)
        self.nl_history = history
        N.check(self.lib, self.lib.px_nl_finish(self.h, s), self.h)
        return history

    def finish_direct(self, stream: int | None = None) -> None:
        s = current_stream_handle() if stream is None else stream
        N.check(self.lib, self.lib.px_finish_direct(self.h, s), self.h)

    def set_adjoint_mode(self, mode: str) -> None:
        """Burgers adjoint formulation (`px_set_adjoint_mode`): "absorbed" (Option A,
        `solve_adjoint_varying`, config 3) or "frozen_span" (the reference's `solve_hybrid`:
        q†_T propagated through the frozen J(ū_p)ᵀ, `hybrid.py:212-237`)."""
        code = {"absorbed": N.PX_ADJOINT_ABSORBED, "frozen_span": N.PX_ADJOINT_FROZEN_SPAN}.get(mode)
        if code is None:
            raise ValueError(f"adjoint mode must be 'absorbed' or 'frozen_span', not {mode!r}")
        N.check(self.lib, self.lib.px_set_adjoint_mode(self.h, code), self.h)
        self._adjoint_mode = mode

    def adjoint_partial(self, stream: int | None = None) -> None:
        self._detach_snapshots()
        s = current_stream_handle() if stream is None else stream
        span = self._adjoint_mode == "frozen_span"
        if not self.spec.system.is_linear and (self.p1 - self.p0 > 1 or self.p0 > 0 or span):
            self.plan_frozen(s)  # no carry for a single absorbed slice (the serial loop)
        N.check(self.lib, self.lib.px_adjoint(self.h, s), self.h)

    def finish_adjoint(self, stream: int | None = None) -> None:
        s = current_stream_handle() if stream is None else stream
        N.check(self.lib, self.lib.px_finish_adjoint(self.h, s), self.h)

    def direct_reduce_fields(self) -> list[int]:
        return [N.PX_FIELD_UT] if self.spec.system.is_linear else []

    @staticmethod
    def adjoint_reduce_fields(want_fields: bool = True) -> list[int]:
        return [N.PX_FIELD_GRAD] + ([N.PX_FIELD_QDAG0, N.PX_FIELD_G] if want_fields else [])


    def plan_frozen(self, stream: int | None = None) -> ChebPlan:
        """Burgers: read the frozen-operator FOV union, plan on the host (cached)."""
        lo, hi, im = self.get(N.PX_FIELD_FROZEN_BOUNDS, stream)
        if not np.all(np.isfinite([lo, hi, im])):  # a non-finite direct trajectory
            raise IntegrationFailure(self.spec.system.spec.T, "non-finite Burgers trajectory")
        region = frozen_region_from_bounds(float(lo), float(hi), float(im))
        cfg = self.spec.expaction
        if not isinstance(cfg, ChebyshevConfig):
            raise ConfigError("the Burgers frozen adjoint uses the Chebyshev action")
        plan = plan_chebyshev(region, self.spec.system.spec.T / self.spec.P, cfg)
        self._set_plan(N.PX_PLAN_FROZEN, plan)
        return plan


    def set_adjoint_terminal(self, qdag_T, stream: int | None = None) -> None:
        self._detach_snapshots()
        s = current_stream_handle() if stream is None else stream
        a = np.ascontiguousarray(qdag_T, dtype=np.float64).reshape(-1)
        if a.size != self.B * self.n:
            raise ValueError("qdag_T must have B·n values")
        N.check(self.lib, self.lib.px_set_adjoint_terminal(self.h, a.ctypes.data, N.PX_MEM_HOST, s), self.h)
        self._keep.append(a)

    def gradient(self, stream: int | None = None, group=None, want_fields: bool = True) -> None:
        """One full direct-adjoint gradient evaluation, enqueued on ``stream``."""
        self._detach_snapshots()
        s = current_stream_handle() if stream is None else stream
        if self.spec.world == 1 and self.spec.system.is_linear:
            N.check(self.lib, self.lib.px_gradient(self.h, s), self.h)
            return
        if self.spec.world == 1:
            self.direct_partial(s)
            self.finish_direct(s)
            self.adjoint_partial(s)
            self.finish_adjoint(s)
            return
        distributed_gradient(self, s, group, want_fields)

    def results(self, stream: int | None = None, fields: bool = True) -> dict:
        J = self.get(N.PX_FIELD_J, stream)
        if not np.all(np.isfinite(J)):
            raise IntegrationFailure(self.spec.system.spec.T, "non-finite objective")
        out = {"J": J, "grad": self.get(N.PX_FIELD_GRAD, stream).reshape(self.B, self.K)}
        if fields:
            out["uT"] = self.get(N.PX_FIELD_UT, stream).reshape(self.B, self.n)
            out["qdag0"] = self.get(N.PX_FIELD_QDAG0, stream).reshape(self.B, self.n)
            out["G"] = self.get(N.PX_FIELD_G, stream).reshape(self.B, self.n)
        return out

    def snapshot(self, field: int, shape):
        """A result field read to the host on first use (`optimization.DeviceField`): it views
        the native buffer and is copied on the device only if this engine is about to overwrite
        it while the field is still referenced (copy-on-write, `_detach_snapshots`); a host
        array when torch/CUDA is unavailable."""
        import weakref

        from .optimization import DeviceField
        torch = _torch()
        if torch is None or not torch.cuda.is_available():
            return self.get(field).reshape(shape)
        f = DeviceField(self.device_view(field), shape, live=True)
        self._snapshots = [r for r in getattr(self, "_snapshots", []) if r() is not None]
        self._snapshots.append(weakref.ref(f))
        return f

    def _detach_snapshots(self) -> None:
        for r in getattr(self, "_snapshots", []):
            f = r()
            if f is not None:
                f.detach()
        self._snapshots = []

    def close(self) -> None:
        self._detach_snapshots()
        if getattr(self, "h", None):
            self.lib.px_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
