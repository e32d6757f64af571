"""CPU oracle, config mode — TEST INFRASTRUCTURE ONLY.

This module is the checker for the CUDA path. Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline / ``--impl reference``
legs may import it; the product package never does (and has no CPU fallback).

It is a plain numpy restatement of the reference's Paraexp structure with the
BASELINE configs' numerics (fixed-step classical RK4, Chebyshev/Krylov exponential
actions, terminal objective, time-constant Fourier control). Structure followed:

* absorbed initial condition, per-slice zero-data inhomogeneous solves, homogeneous
  propagation, superposition — `pkg/src/paradjoint/paraexp.py:187-248`;
* absorbed final condition, reflected time σ = T_p + T_{p+1} − t, chains P → 0 —
  `paraexp.py:256-326`; time-varying operator + per-slice frozen operator —
  `paraexp.py:329-353`, `systems.py:64-97`;
* Burgers: serial direct sweep keeping the trajectory (`hybrid.py:185-191`),
  matrix-free Jᵀ(u)y (`problems.py:316-343`, V ≡ 0), linear interpolation of the
  stored trajectory (`timestepping.py:64-75`), trapezoid-averaged frozen
  linearisation (`problems.py:346-366`);
* objective/gradient conventions: unweighted inner products (`PAPER.md:149-155`),
  ∂J/∂c_k = ⟨φ_k, ∫q† dt⟩ (control-to-state map ∂N/∂c_k = φ_k).

Homogeneous formulations: ``chains`` is the reference's
neighbour form (each slice end propagated separately, `paraexp.py:207-217`);
``scan`` is the summed-chain carry D_{p+1} = exp(ΔA)·D_p + v_p (equal by
linearity, P−1 actions); ``blockscan`` with G ranks is scan per contiguous block
plus one long action per block (the multi-GPU form). The GPU executes the same
operation sequence as ``scan``/``blockscan`` so parity is at rounding level.

The exponential-action plans (degree, substeps, coefficients) are inputs — built
by the product's host planner, validated independently here against FFT-exact
circulant propagators (tests/test_oracle.py).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from paper_2004_00546_b200.expaction import ChebPlan, KrylovPlan
from paper_2004_00546_b200.partition import rank_block

from .reference_mode import chains_adjoint, chains_direct

# ---------------------------------------------------------------------------
# Operators
# ---------------------------------------------------------------------------


def stencil_apply(st, u: np.ndarray, nx: int, ny: int) -> np.ndarray:
    """(M u) with coefficients (cc, ce, cw, cn, cs) on a periodic grid, x fastest.

    Same operator as `problems.py:149-152` (central differences, periodic wrap).
    """
    cc, ce, cw, cn, cs = st
    shp = u.shape
    U = u.reshape(shp[:-1] + (ny, nx))
    out = cc * U + ce * np.roll(U, -1, axis=-1) + cw * np.roll(U, 1, axis=-1)
    if ny > 1:
        out = out + cn * np.roll(U, -1, axis=-2) + cs * np.roll(U, 1, axis=-2)
    return out.reshape(shp)


def dx_central(u: np.ndarray, h: float) -> np.ndarray:
    return (np.roll(u, -1, axis=-1) - np.roll(u, 1, axis=-1)) / (2.0 * h)


def burgers_rhs(u, f, D, h):
    """−u∘Dx u + D·L u + f (`problems.py:177-185` with V ≡ 0, time-constant f)."""
    lap = (np.roll(u, -1, axis=-1) - 2.0 * u + np.roll(u, 1, axis=-1)) / (h * h)
    return -u * dx_central(u, h) + D * lap + f


def burgers_adjoint_apply(u, y, D, h):
    """J(u)ᵀy = Dx(u∘y) − (Dx u)∘y + D·L y (`problems.py:316-343`, V ≡ 0)."""
    lap = (np.roll(y, -1, axis=-1) - 2.0 * y + np.roll(y, 1, axis=-1)) / (h * h)
    return dx_central(u * y, h) - dx_central(u, h) * y + D * lap


def _split2(q, nx, ny):
    """(…, 2n) state → U, V as (…, ny, nx) grids (x fastest; `problems.py:170-174`)."""
    n = nx * ny
    shp = q.shape[:-1]
    return q[..., :n].reshape(shp + (ny, nx)), q[..., n:].reshape(shp + (ny, nx))


def _d2(W, hx, hy):
    """Periodic central Dx, Dy and the 5-point Laplacian of a (…, ny, nx) grid (`problems.py:98-134`)."""
    e, w = np.roll(W, -1, axis=-1), np.roll(W, 1, axis=-1)
    n_, s_ = np.roll(W, -1, axis=-2), np.roll(W, 1, axis=-2)
    return (e - w) / (2.0 * hx), (n_ - s_) / (2.0 * hy), (e - 2.0 * W + w) / (hx * hx) + (n_ - 2.0 * W + s_) / (hy * hy)


def burgers2d_rhs(q, f, D, hx, hy, nx, ny):
    """Two-field viscous Burgers rhs (`problems.py:177-186`): −U∂xU − V∂yU + D∇²U + f_U and the
    same for V; ``q`` and ``f`` are (…, 2n) with the U block first."""
    U, V = _split2(q, nx, ny)
    dUx, dUy, lU = _d2(U, hx, hy)
    dVx, dVy, lV = _d2(V, hx, hy)
    ru = -U * dUx - V * dUy + D * lU
    rv = -U * dVx - V * dVy + D * lV
    shp = q.shape[:-1]
    return np.concatenate([ru.reshape(shp + (-1,)), rv.reshape(shp + (-1,))], axis=-1) + f


def burgers2d_adjoint_apply(q, y, D, hx, hy, nx, ny):
    """J(q)ᵀy of the two-field system (`problems.py:316-343`):
    out_a = ∂x(U a) + ∂y(V a) − (∂xU) a − (∂xV) b + D∇²a,
    out_b = ∂x(U b) + ∂y(V b) − (∂yU) a − (∂yV) b + D∇²b."""
    U, V = _split2(q, nx, ny)
    a, b = _split2(y, nx, ny)
    dUx, dUy, _ = _d2(U, hx, hy)
    dVx, dVy, _ = _d2(V, hx, hy)
    dxUa, _, la = _d2(U * a, hx, hy)
    _, dyVa, _ = _d2(V * a, hx, hy)
    dxUb, _, _ = _d2(U * b, hx, hy)
    _, dyVb, _ = _d2(V * b, hx, hy)
    _, _, la = _d2(a, hx, hy)
    _, _, lb = _d2(b, hx, hy)
    oa = dxUa + dyVa - dUx * a - dVx * b + D * la
    ob = dxUb + dyVb - dUy * a - dVy * b + D * lb
    shp = np.broadcast_shapes(q.shape[:-1], y.shape[:-1])
    return np.concatenate([oa.reshape(shp + (-1,)), ob.reshape(shp + (-1,))], axis=-1)


def burgers2d_advection(q, hx, hy, nx, ny):
    """N(q) = (−U∂xU − V∂yU, −U∂xV − V∂yV) (`problems.py:189-195`)."""
    U, V = _split2(q, nx, ny)
    dUx, dUy, _ = _d2(U, hx, hy)
    dVx, dVy, _ = _d2(V, hx, hy)
    shp = q.shape[:-1]
    return np.concatenate([(-U * dUx - V * dUy).reshape(shp + (-1,)), (-U * dVx - V * dVy).reshape(shp + (-1,))],
                          axis=-1)


def burgers2d_advection_jacobian_apply(qbar, y, hx, hy, nx, ny):
    """(∂N/∂q at q̄)·y (`problems.py:213-287`): (−Ū∂x a − V̄∂y a − (∂xŪ)a − (∂yŪ)b,
    −Ū∂x b − V̄∂y b − (∂xV̄)a − (∂yV̄)b)."""
    U, V = _split2(qbar, nx, ny)
    a, b = _split2(y, nx, ny)
    dUx, dUy, _ = _d2(U, hx, hy)
    dVx, dVy, _ = _d2(V, hx, hy)
    dax, day, _ = _d2(a, hx, hy)
    dbx, dby, _ = _d2(b, hx, hy)
    oa = -U * dax - V * day - dUx * a - dUy * b
    ob = -U * dbx - V * dby - dVx * a - dVy * b
    shp = np.broadcast_shapes(qbar.shape[:-1], y.shape[:-1])
    return np.concatenate([oa.reshape(shp + (-1,)), ob.reshape(shp + (-1,))], axis=-1)


def laplacian2d(q, D, hx, hy, nx, ny):
    U, V = _split2(q, nx, ny)
    shp = q.shape[:-1]
    return D * np.concatenate([_d2(U, hx, hy)[2].reshape(shp + (-1,)), _d2(V, hx, hy)[2].reshape(shp + (-1,))], axis=-1)


def burgers_ops(nx, D, ny=None, hy=None):
    """(rhs(u, f), adj(u, y), n) of the Burgers testbed: 1D one-field (ny None) or the
    reference's 2D two-field system (state length 2·nx·ny)."""
    hx = 2.0 * np.pi / nx
    if ny is None:
        return (lambda u, f: burgers_rhs(u, f, D, hx)), (lambda u, y: burgers_adjoint_apply(u, y, D, hx)), nx
    hy = 2.0 * np.pi / ny if hy is None else hy
    return ((lambda u, f: burgers2d_rhs(u, f, D, hx, hy, nx, ny)),
            (lambda u, y: burgers2d_adjoint_apply(u, y, D, hx, hy, nx, ny)), 2 * nx * ny)


# ---------------------------------------------------------------------------
# Steppers and exponential actions
# ---------------------------------------------------------------------------


def rk4_linear(apply, g, h: float, nsteps: int, want_z: bool = False):
    """Zero-data classical RK4 for y' = M y + g; optionally z = ∫y (RK4-consistent).

    z is RK4 applied to the augmented system (y, z)' = (M y + g, y).
    """
    y = np.zeros_like(g)
    z = np.zeros_like(g) if want_z else None
    for _ in range(nsteps):
        k1 = apply(y) + g
        Y2 = y + (0.5 * h) * k1
        k2 = apply(Y2) + g
        Y3 = y + (0.5 * h) * k2
        k3 = apply(Y3) + g
        Y4 = y + h * k3
        k4 = apply(Y4) + g
        if want_z:
            z = z + (h / 6.0) * (y + 2.0 * Y2 + 2.0 * Y3 + Y4)
        y = y + (h / 6.0) * (k1 + 2.0 * k2 + 2.0 * k3 + k4)
    return y, z


def cheb_action(apply, plan: ChebPlan, v: np.ndarray, phi: np.ndarray | None = None):
    """exp(span·M)v by substeps of the planned Chebyshev series; when ``phi`` is
    given, adds span·φ₁(span·M)v = Σ_j exp(jτ_s M)(τ_s φ₁(τ_s M) y_j) into it."""
    c0, d, sigma = plan.center, plan.scale, float(plan.sigma)
    be, bp = plan.coef_exp, plan.coef_phi
    two_over = 2.0 / d
    y = v
    for _ in range(plan.substeps):
        u_prev = y
        acc = be[0] * u_prev
        pacc = bp[0] * u_prev if phi is not None else None
        u_cur = (apply(u_prev) - c0 * u_prev) / d
        acc = acc + be[1] * u_cur
        if phi is not None:
            pacc = pacc + bp[1] * u_cur
        for k in range(2, plan.degree + 1):
            u_next = two_over * (apply(u_cur) - c0 * u_cur) + sigma * u_prev
            u_prev, u_cur = u_cur, u_next
            acc = acc + be[k] * u_cur
            if phi is not None:
                pacc = pacc + bp[k] * u_cur
        if phi is not None:
            phi += pacc
        y = acc
    return y


def expm_taylor(A: np.ndarray) -> np.ndarray:
    """exp(A) by scaling and squaring with a degree-18 Taylor polynomial."""
    nrm = float(np.max(np.sum(np.abs(A), axis=0))) if A.size else 0.0
    sq = 0 if nrm <= 0.5 else int(np.ceil(np.log2(nrm / 0.5)))
    B = A / (2.0 ** sq)
    n = A.shape[0]
    E = np.eye(n)
    for k in range(18, 0, -1):
        E = np.eye(n) + (B @ E) / k
    for _ in range(sq):
        E = E @ E
    return E


KRYLOV_BREAKDOWN = 1e-13


def krylov_action(apply, plan: KrylovPlan, v: np.ndarray, phi: np.ndarray | None = None):
    """exp(span·M)v by substeps of m-step Arnoldi (CGS2) + small augmented expm.

    Per substep: y_{j+1} = β V_m e^{τH_m} e_1 and φ += β V_m τφ₁(τH_m) e_1, both
    read off exp([[τH_m, τe_1], [0, 0]]). Happy breakdown (h_{j+1,j} ≤
    1e-13·β_0-scaled) truncates the basis.
    """
    m = plan.m
    tau = plan.span / plan.substeps
    y = v
    for _ in range(plan.substeps):
        beta = float(np.sqrt(np.dot(y, y)))
        if beta == 0.0:
            continue
        V = np.zeros((m + 1, y.size))
        H = np.zeros((m + 1, m))
        V[0] = y / beta
        meff = m
        for j in range(m):
            w = apply(V[j])
            h1 = V[: j + 1] @ w
            w = w - V[: j + 1].T @ h1
            h2 = V[: j + 1] @ w
            w = w - V[: j + 1].T @ h2
            H[: j + 1, j] = h1 + h2
            nrm = float(np.sqrt(np.dot(w, w)))
            H[j + 1, j] = nrm
            if nrm <= KRYLOV_BREAKDOWN * max(1.0, float(np.max(np.abs(H[: j + 2, j])))):
                meff = j + 1
                break
            V[j + 1] = w / nrm
        Ha = np.zeros((meff + 1, meff + 1))
        Ha[:meff, :meff] = tau * H[:meff, :meff]
        Ha[0, meff] = tau
        E = expm_taylor(Ha)
        ce = beta * E[:meff, 0]
        cp = beta * E[:meff, meff]
        if phi is not None:
            phi += cp @ V[:meff]
        y = ce @ V[:meff]
    return y


def exp_action(apply, plan, v, phi=None):
    if isinstance(plan, KrylovPlan):
        if v.ndim == 1:
            return krylov_action(apply, plan, v, phi)
        # one Arnoldi process per batch member (the GPU batches them in one grid)
        out = np.empty_like(v)
        for b in range(v.shape[0]):
            out[b] = krylov_action(apply, plan, v[b], None if phi is None else phi[b])
        return out
    return cheb_action(apply, plan, v, phi)


# ---------------------------------------------------------------------------
# Linear advection–diffusion gradient (configs 1, 2, 4, 5)
# ---------------------------------------------------------------------------


@dataclass
class OracleResult:
    J: np.ndarray                 # (B,)
    grad: np.ndarray              # (B, K)
    uT: np.ndarray                # (B, n)
    qdag0: np.ndarray             # (B, n)
    G: np.ndarray                 # (B, n)  ∫ q† dt
    u_bnd: np.ndarray | None = None   # (B, P+1, n) direct boundary states (scan only)
    extras: dict = field(default_factory=dict)


def _as_batch(a, n):
    a = np.asarray(a, dtype=np.float64)
    return a.reshape(-1, n) if a.ndim > 1 else a[None, :]


def _block_bounds(P, world, sizes=None, mirrored=False):
    """Contiguous slice blocks: `rank_block` (equal) or explicit sizes; the adjoint of the GPU's
    local blocks uses the mirrored partition (engine._block_sizes)."""
    if sizes is None:
        return [rank_block(P, r, world) for r in range(world)]
    sz = list(sizes)[::-1] if mirrored else list(sizes)
    out, q = [], 0
    for s_ in sz:
        out.append((q, q + s_))
        q += s_
    return out


def linear_gradient(grid_nx, grid_ny, A, basis, T, P, nsteps, u0, u_target, ctrl,
                    plan_slice, plan_long_direct=None, plan_long_adjoint=None,
                    formulation: str = "scan", world: int = 1, want_boundary=False, qdag_T=None,
                    block_sizes=None):
    """One Paraexp direct-adjoint gradient for the linear testbed (App. B of SURVEY).

    ``A`` stencil tuple; ``basis`` ModeBasis; ``ctrl`` (B, K). ``plan_long_*``:
    callables span → plan for the blockscan long spans (world > 1). ``qdag_T``
    overrides the adjoint's terminal condition (a checkpointed segment's carried q†,
    `checkpointing.py:192-251`); default u(T) − u_target.
    """
    nx, ny = grid_nx, grid_ny
    n = nx * ny
    ctrl = np.atleast_2d(np.asarray(ctrl, dtype=np.float64))
    B = ctrl.shape[0]
    u0 = _as_batch(u0, n)
    u0 = np.broadcast_to(u0, (B, n))
    ut = np.broadcast_to(_as_batch(u_target, n), (B, n))
    AT = tuple(np.asarray(A)[[0, 2, 1, 4, 3]])
    applyA = lambda u: stencil_apply(A, u, nx, ny)
    applyAT = lambda u: stencil_apply(AT, u, nx, ny)
    delta = T / P
    h = delta / nsteps

    f = basis.field(ctrl)                        # (B, n)
    g = applyA(u0) + f                           # absorbed IC source (`paraexp.py:239-242`)
    # every slice solves the same zero-data problem (time-constant source);
    # the checker computes it once, the GPU computes all P of them.
    v_end, _ = rk4_linear(applyA, g, h, nsteps)

    u_bnd = None
    bounds = T * np.arange(P + 1) / P
    if formulation == "chains":
        # the reference's neighbour-chain structure (reference_mode.chains_direct,
        # pinned to `solve_direct_linear`) with RK4 slices and Chebyshev chains
        zero_end = np.stack([np.zeros_like(v_end), v_end])
        pieces = chains_direct(
            bounds, u0, lambda p: (bounds[p:p + 2], zero_end),
            lambda p, start, m: (lambda e: (e, e[None]))(exp_action(applyA, plan_slice, start)),
            lambda p: bounds[p:p + 2])
        uT = pieces[-1][1][-1]
    elif formulation == "scan" and world == 1:
        D = np.zeros_like(v_end)
        if want_boundary:
            u_bnd = np.empty((B, P + 1, n))
            u_bnd[:, 0] = u0
        for p in range(P):
            D = v_end.copy() if p == 0 else exp_action(applyA, plan_slice, D) + v_end
            if want_boundary:
                u_bnd[:, p + 1] = u0 + D
        uT = u0 + D
    else:  # blockscan over `world` contiguous blocks, summed as an allreduce would
        partial = np.zeros_like(v_end)
        for p0, p1 in _block_bounds(P, world, block_sizes):
            D = np.zeros_like(v_end)
            for p in range(p0, p1):
                D = v_end.copy() if p == p0 else exp_action(applyA, plan_slice, D) + v_end
            if p1 < P:
                D = exp_action(applyA, plan_long_direct((P - p1) * delta), D)
            partial = partial + D
        uT = u0 + partial

    qT = uT - ut
    J = 0.5 * np.sum(qT * qT, axis=1)
    if qdag_T is not None:
        qT = np.broadcast_to(_as_batch(qdag_T, n), (B, n)).copy()

    # adjoint: w' = Aᵀ(w + q†_T), zero data, per slice; z = ∫w
    gadj = applyAT(qT)
    w_end, z = rk4_linear(applyAT, gadj, h, nsteps, want_z=True)
    if formulation == "chains":
        # reference_mode.chains_adjoint (pinned to `solve_adjoint_linear`); the φ₁
        # accumulator collects ∫ of every homogeneous chain piece
        Gh = np.zeros_like(w_end)
        zero_end = np.stack([np.zeros_like(w_end), w_end])
        pieces = chains_adjoint(
            bounds, qT, lambda p: (bounds[p:p + 2], zero_end),
            lambda p, start, m: (lambda e: (e, e[None]))(exp_action(applyAT, plan_slice, start, Gh)),
            lambda p: bounds[p:p + 2])
        qdag0 = pieces[0][1][0]
        G = T * qT + P * z + Gh
    elif formulation == "scan" and world == 1:
        C = np.zeros_like(w_end)
        Gh = np.zeros_like(w_end)
        for p in range(P - 1, -1, -1):
            C = w_end.copy() if p == P - 1 else exp_action(applyAT, plan_slice, C, Gh) + w_end
        qdag0 = qT + C
        G = T * qT + P * z + Gh
    else:
        qd = np.zeros_like(w_end)
        Gh = np.zeros_like(w_end)
        for p0, p1 in _block_bounds(P, world, block_sizes, mirrored=True):
            C = np.zeros_like(w_end)
            Gr = np.zeros_like(w_end)
            for p in range(p1 - 1, p0 - 1, -1):
                C = w_end.copy() if p == p1 - 1 else exp_action(applyAT, plan_slice, C, Gr) + w_end
            if p0 > 0:
                C = exp_action(applyAT, plan_long_adjoint(p0 * delta), C, Gr)
            qd = qd + C
            Gh = Gh + (p1 - p0) * z + Gr
        qdag0 = qT + qd
        G = T * qT + Gh
    grad = basis.project(G)
    return OracleResult(J=J, grad=grad, uT=uT, qdag0=qdag0, G=G, u_bnd=u_bnd,
                        extras={"v_end": v_end, "w_end": w_end, "z": z})


# ---------------------------------------------------------------------------
# Burgers (config 3): serial direct + Paraexp adjoint with frozen slices
# ---------------------------------------------------------------------------


def burgers_direct(u0, f, D, h_grid, h, nsteps_total):
    """Serial classical RK4 keeping every node (the HBM trajectory)."""
    traj = np.empty((nsteps_total + 1,) + u0.shape)
    u = u0.copy()
    traj[0] = u
    for i in range(nsteps_total):
        k1 = burgers_rhs(u, f, D, h_grid)
        k2 = burgers_rhs(u + (0.5 * h) * k1, f, D, h_grid)
        k3 = burgers_rhs(u + (0.5 * h) * k2, f, D, h_grid)
        k4 = burgers_rhs(u + h * k3, f, D, h_grid)
        u = u + (h / 6.0) * (k1 + 2.0 * k2 + 2.0 * k3 + k4)
        traj[i + 1] = u
    return traj


def slice_means(traj, P, nsteps):
    """Trapezoid-weighted mean of each slice's nodes (`problems.py:346-366`)."""
    w = np.ones(nsteps + 1)
    w[0] = w[-1] = 0.5
    w /= nsteps
    return np.stack([np.tensordot(w, traj[p * nsteps: (p + 1) * nsteps + 1], axes=(0, 0))
                     for p in range(P)])


def burgers_gradient(nx, D, basis, T, P, nsteps, u0, u_target, ctrl, plan_for_region,
                     region_fn, world: int = 1, traj=None, qdag_T=None, adjoint: str = "absorbed"):
    """Config 3 (Option A of SURVEY §8(c)): absorbed final condition, exact Jᵀ(u(t))
    in the inhomogeneous solves, frozen J(ū_p)ᵀ in the homogeneous ones.

    ``adjoint="frozen_span"``: the reference's `solve_hybrid` (Option B,
    `hybrid.py:194-237`): the inhomogeneous solves start from zero terminal data
    (`hybrid.py:194-203`) and, with the terminal objective's zero adjoint source, vanish;
    q† is q†_T propagated over [T, 0] through the frozen J(ū_p)ᵀ slice by slice
    (`propagate_span`, `hybrid.py:212-225`; the final span `hybrid.py:232-233`), and
    ∫q† dt is the φ₁ series of the same actions."""
    n = nx
    hg = 2.0 * np.pi / nx
    ctrl = np.atleast_2d(np.asarray(ctrl, dtype=np.float64))
    B = ctrl.shape[0]
    u0 = np.broadcast_to(_as_batch(u0, n), (B, n)).copy()
    ut = np.broadcast_to(_as_batch(u_target, n), (B, n))
    delta = T / P
    h = delta / nsteps
    f = basis.field(ctrl)
    if traj is None:   # serial direct sweep; Algorithm 2 passes its converged iterate
        traj = burgers_direct(u0, f, D, hg, h, P * nsteps)      # (S+1, B, n)
    uT = traj[-1]
    qT = uT - ut
    J = 0.5 * np.sum(qT * qT, axis=1)
    if qdag_T is not None:   # checkpointed segment: carried q† (`checkpointing.py:192-251`)
        qT = np.broadcast_to(_as_batch(qdag_T, n), (B, n)).copy()

    ubar = slice_means(traj, P, nsteps)                          # (P, B, n)
    region = region_fn(ubar)
    plan = plan_for_region(region, delta)

    if adjoint == "frozen_span":
        C = qT.copy()
        Gh = np.zeros((B, n))
        for p in range(P - 1, -1, -1):
            ub = ubar[p]
            C = exp_action(lambda y, ub=ub: burgers_adjoint_apply(ub, y, D, hg), plan, C, Gh)
        grad = basis.project(Gh)
        return OracleResult(J=J, grad=grad, uT=uT, qdag0=C, G=Gh,
                            extras={"traj": traj, "ubar": ubar, "plan": plan})
    if adjoint != "absorbed":
        raise ValueError(adjoint)

    w_end = np.empty((P, B, n))
    zsum = np.zeros((B, n))
    for p in range(P):
        w = np.zeros((B, n))
        z = np.zeros((B, n))
        top = (p + 1) * nsteps
        for i in range(nsteps):
            ua = traj[top - i]
            ub = traj[top - i - 1]
            um = 0.5 * ua + 0.5 * ub
            k1 = burgers_adjoint_apply(ua, w + qT, D, hg)
            Y2 = w + (0.5 * h) * k1
            k2 = burgers_adjoint_apply(um, Y2 + qT, D, hg)
            Y3 = w + (0.5 * h) * k2
            k3 = burgers_adjoint_apply(um, Y3 + qT, D, hg)
            Y4 = w + h * k3
            k4 = burgers_adjoint_apply(ub, Y4 + qT, D, hg)
            z = z + (h / 6.0) * (w + 2.0 * Y2 + 2.0 * Y3 + Y4)
            w = w + (h / 6.0) * (k1 + 2.0 * k2 + 2.0 * k3 + k4)
        w_end[p] = w
        zsum += z

    def frozen(p):
        ub = ubar[p]
        return lambda y: burgers_adjoint_apply(ub, y, D, hg)

    qd = np.zeros((B, n))
    Gh = np.zeros((B, n))
    for r in range(world):
        p0, p1 = rank_block(P, r, world)
        C = np.zeros((B, n))
        for p in range(p1 - 1, p0 - 1, -1):
            C = w_end[p].copy() if p == p1 - 1 else exp_action(frozen(p), plan, C, Gh) + w_end[p]
        for p in range(p0 - 1, -1, -1):       # carry through earlier ranks' frozen slices
            C = exp_action(frozen(p), plan, C, Gh)
        qd = qd + C
    qdag0 = qT + qd
    G = T * qT + zsum + Gh
    grad = basis.project(G)
    return OracleResult(J=J, grad=grad, uT=uT, qdag0=qdag0, G=G,
                        extras={"traj": traj, "ubar": ubar, "plan": plan, "w_end": w_end})


# ---------------------------------------------------------------------------
# Per-rank partials with the C ABI's conventions (for the gloo tests of the
# product's multi-rank orchestration, engine.distributed_gradient)
# ---------------------------------------------------------------------------


class OracleRank:
    """A CPU stand-in for one rank's ParaexpEngine: same phase methods and field
    buffers (torch CPU tensors), computed with the oracle's block-scan pieces."""

    FIELDS = ("J", "GRAD", "UT", "QDAG0", "G")

    def __init__(self, nx, ny, A, basis, T, P, nsteps, u0, u_target, ctrl, plan_slice, plan_long, rank, world):
        import torch
        self.nx, self.ny, self.T, self.P, self.nsteps = nx, ny, T, P, nsteps
        self.A = tuple(A)
        self.AT = tuple(np.asarray(A)[[0, 2, 1, 4, 3]])
        self.basis = basis
        n = nx * ny
        self.ctrl = np.atleast_2d(np.asarray(ctrl, dtype=np.float64))
        B = self.ctrl.shape[0]
        self.u0 = np.broadcast_to(_as_batch(u0, n), (B, n))
        self.ut = np.broadcast_to(_as_batch(u_target, n), (B, n))
        self.plan_slice, self.plan_long = plan_slice, plan_long
        self.p0, self.p1 = rank_block(P, rank, world)
        from types import SimpleNamespace
        self.spec = SimpleNamespace(rank=rank, world=world)  # the engine's (rank, world) for fail-fast
        self.buf = {k: torch.zeros(B * (basis.K if k == "GRAD" else (1 if k == "J" else n)), dtype=torch.float64)
                    for k in self.FIELDS}
        self.B, self.n = B, n

    def _np(self, k):
        return self.buf[k].numpy().reshape(self.B, -1)

    def view(self, k):
        return self.buf[k]

    @staticmethod
    def direct_reduce_fields():
        return ["UT"]

    @staticmethod
    def adjoint_reduce_fields(want_fields=True):
        return ["GRAD"] + (["QDAG0", "G"] if want_fields else [])

    def direct_partial(self, stream=None):
        applyA = lambda u: stencil_apply(self.A, u, self.nx, self.ny)
        h = self.T / self.P / self.nsteps
        g = applyA(self.u0) + self.basis.field(self.ctrl)
        v_end, _ = rk4_linear(applyA, g, h, self.nsteps)
        D = np.zeros_like(v_end)
        for p in range(self.p0, self.p1):
            D = v_end.copy() if p == self.p0 else exp_action(applyA, self.plan_slice, D) + v_end
        if self.p1 < self.P:
            D = exp_action(applyA, self.plan_long((self.P - self.p1) * self.T / self.P), D)
        self._np("UT")[:] = D

    def finish_direct(self, stream=None):
        uT = self._np("UT")
        uT += self.u0
        self.qT = uT - self.ut
        self._np("J")[:, 0] = 0.5 * np.sum(self.qT * self.qT, axis=1)

    def adjoint_partial(self, stream=None):
        applyAT = lambda u: stencil_apply(self.AT, u, self.nx, self.ny)
        h = self.T / self.P / self.nsteps
        w_end, z = rk4_linear(applyAT, applyAT(self.qT), h, self.nsteps, want_z=True)
        C = np.zeros_like(w_end)
        Gr = (self.p1 - self.p0) * z
        for p in range(self.p1 - 1, self.p0 - 1, -1):
            C = w_end.copy() if p == self.p1 - 1 else exp_action(applyAT, self.plan_slice, C, Gr) + w_end
        if self.p0 > 0:
            C = exp_action(applyAT, self.plan_long(self.p0 * self.T / self.P), C, Gr)
        self._np("QDAG0")[:] = C
        self._np("G")[:] = Gr
        self._np("GRAD")[:] = self.basis.project(Gr)

    def finish_adjoint(self, stream=None):
        self._np("QDAG0")[:] += self.qT
        self._np("G")[:] += self.T * self.qT
        self._np("GRAD")[:] += self.T * self.basis.project(self.qT)


# ---------------------------------------------------------------------------
# Algorithm 2: iterative Jacobian-augmented Paraexp direct solve (Burgers)
# ---------------------------------------------------------------------------


def jac_apply(ubar, y, D, h):
    """J(ū)·y = D·L y − ū∘Dx y − (Dx ū)∘y (full Burgers linearisation, V ≡ 0)."""
    lap = (np.roll(y, -1, axis=-1) - 2.0 * y + np.roll(y, 1, axis=-1)) / (h * h)
    return D * lap - ubar * dx_central(y, h) - dx_central(ubar, h) * y


def burgers_iterative_direct(nx, D, basis, T, P, nsteps, u0, ctrl, plan_for_region, region_fn, eps,
                             max_iter=25, min_iter=2):
    """`solve_direct_nonlinear` (`nonlinear.py:69-194`) with the configs' numerics.

    Iterate Q (all RK4 nodes, constant u0 initially). Each sweep: ū_p = trapezoid
    slice means of Q; per slice the linear problem y' = J(ū_p)y + s(t),
    s = D·L u0 + f − Q∘Dx Q + ū_p∘Dx(Q − u0) + (Dx ū_p)(Q − u0) (i.e.
    A·q0 + f + N(Q) − J̄_p(Q − q0), `nonlinear.py:113-116`), y(T_p) = 0, RK4 with Q
    linearly interpolated at the stages; summed-chain carry D_{p+1} =
    exp(Δ J(ū_p))D_p + y_p(end); new iterate q0 + y_p(kh) + exp(kh J(ū_p))D_p at
    every node (h-width actions); stop when max_p relative L2 change < eps and at
    least min_iter sweeps ran (`nonlinear.py:137-146`).
    """
    n = nx
    hg = 2.0 * np.pi / nx
    ctrl = np.atleast_2d(np.asarray(ctrl, dtype=np.float64))
    B = ctrl.shape[0]
    u0 = np.broadcast_to(_as_batch(u0, n), (B, n)).copy()
    delta = T / P
    h = delta / nsteps
    f = basis.field(ctrl)
    S = P * nsteps
    Q = np.broadcast_to(u0, (S + 1, B, n)).copy()
    lapu0 = D * (np.roll(u0, -1, axis=-1) - 2.0 * u0 + np.roll(u0, 1, axis=-1)) / (hg * hg)
    history = []
    for it in range(1, max_iter + 1):
        ubar = slice_means(Q, P, nsteps)
        region = region_fn(ubar)
        plan_s = plan_for_region(region, delta)
        plan_h = plan_for_region(region, h)
        Qn = np.empty_like(Q)
        y_end = np.empty((P, B, n))
        for p in range(P):
            ub = ubar[p]

            def src(qt):
                dq = qt - u0
                return lapu0 + f - qt * dx_central(qt, hg) + ub * dx_central(dq, hg) + dx_central(ub, hg) * dq

            y = np.zeros((B, n))
            for k in range(nsteps):
                qa = Q[p * nsteps + k]
                qb = Q[p * nsteps + k + 1]
                qm = 0.5 * qa + 0.5 * qb
                k1 = jac_apply(ub, y, D, hg) + src(qa)
                k2 = jac_apply(ub, y + (0.5 * h) * k1, D, hg) + src(qm)
                k3 = jac_apply(ub, y + (0.5 * h) * k2, D, hg) + src(qm)
                k4 = jac_apply(ub, y + h * k3, D, hg) + src(qb)
                y = y + (h / 6.0) * (k1 + 2.0 * k2 + 2.0 * k3 + k4)
                if k + 1 < nsteps:
                    Qn[p * nsteps + k + 1] = u0 + y
            y_end[p] = y
        # summed-chain carry through the per-slice operators
        Dc = np.zeros((P + 1, B, n))
        for p in range(P):
            op = lambda v, ub=ubar[p]: jac_apply(ub, v, D, hg)
            Dc[p + 1] = (y_end[p].copy() if p == 0 else exp_action(op, plan_s, Dc[p]) + y_end[p])
        for p in range(P):
            op = lambda v, ub=ubar[p]: jac_apply(ub, v, D, hg)
            Qn[p * nsteps] = u0 + Dc[p]
            H = Dc[p]
            for k in range(1, nsteps):
                H = exp_action(op, plan_h, H)
                Qn[p * nsteps + k] += H
        Qn[S] = u0 + Dc[P]
        # max over slices (and members) of the relative L2 change on the slice nodes
        err = 0.0
        for p in range(P):
            a = Qn[p * nsteps:(p + 1) * nsteps + 1]
            b = Q[p * nsteps:(p + 1) * nsteps + 1]
            for m in range(B):
                num = float(np.sqrt(np.sum((a[:, m] - b[:, m]) ** 2)))
                den = float(np.sqrt(np.sum(b[:, m] ** 2)))
                err = max(err, num / den if den > 0 else num)
        history.append(err)
        Q = Qn
        if err < eps and it >= min_iter:
            return Q, it, history
    raise RuntimeError(f"no convergence after {max_iter} sweeps: {history}")


def burgers2d_iterative_direct(nx, ny, D, T, P, nsteps, u0, f, law, plans_for, eps, max_iter=25, min_iter=2):
    """`solve_direct_nonlinear` (`nonlinear.py:69-194`) on the reference's two-field 2D Burgers
    system with the forcing f·θ(t) and the configs' numerics — the 2D form of
    `burgers_iterative_direct`: iterate Q on all RK4 nodes (constant u0 initially); per sweep the
    slice means q̄_p, per slice y' = (D∇² + J̄_p)y + s(t), s = D∇²u0 + θ(t)f + N(Q) − J̄_p(Q − u0)
    (J̄_p = ∂N/∂q at q̄_p, `nonlinear.py:113-116`), y(T_p) = 0, classical RK4 with Q linearly
    interpolated at the stages; summed-chain carry D_{p+1} = exp(Δ(D∇² + J̄_p))D_p + y_p(end); the
    new iterate u0 + y_p(kh) + exp(kh(D∇² + J̄_p))D_p on every node; stop when the largest per-slice
    relative L2 change is below eps after at least min_iter sweeps. ``plans_for(qbar)`` returns
    (slice-width plan, step-width plan). Returns (Q, sweeps, history)."""
    hx, hy = 2.0 * np.pi / nx, 2.0 * np.pi / ny
    n2 = 2 * nx * ny
    f = np.atleast_2d(np.asarray(f, dtype=np.float64))
    B = f.shape[0]
    u0 = np.broadcast_to(_as_batch(u0, n2), (B, n2)).copy()
    delta = T / P
    h = delta / nsteps
    S = P * nsteps
    Q = np.broadcast_to(u0, (S + 1, B, n2)).copy()
    lapu0 = laplacian2d(u0, D, hx, hy, nx, ny)
    jadv = lambda qb, y: burgers2d_advection_jacobian_apply(qb, y, hx, hy, nx, ny)
    jfull = lambda qb, y: jadv(qb, y) + laplacian2d(y, D, hx, hy, nx, ny)
    history = []
    for it in range(1, max_iter + 1):
        qbar = slice_means(Q, P, nsteps)
        plan_s, plan_h = plans_for(qbar)
        Qn = np.empty_like(Q)
        y_end = np.empty((P, B, n2))
        for p in range(P):
            qb_ = qbar[p]

            def src(qt, t):
                return (lapu0 + law_value(law, t) * f + burgers2d_advection(qt, hx, hy, nx, ny) - jadv(qb_, qt - u0))

            y = np.zeros((B, n2))
            for k in range(nsteps):
                node = p * nsteps + k
                t = node * h
                qa, qc = Q[node], Q[node + 1]
                qm = 0.5 * qa + 0.5 * qc
                k1 = jfull(qb_, y) + src(qa, t)
                k2 = jfull(qb_, y + (0.5 * h) * k1) + src(qm, t + 0.5 * h)
                k3 = jfull(qb_, y + (0.5 * h) * k2) + src(qm, t + 0.5 * h)
                k4 = jfull(qb_, y + h * k3) + src(qc, t + h)
                y = y + (h / 6.0) * (k1 + 2.0 * k2 + 2.0 * k3 + k4)
                if k + 1 < nsteps:
                    Qn[node + 1] = u0 + y
            y_end[p] = y
        Dc = np.zeros((P + 1, B, n2))
        for p in range(P):
            op = lambda v, qb_=qbar[p]: jfull(qb_, v)
            Dc[p + 1] = (y_end[p].copy() if p == 0 else exp_action(op, plan_s, Dc[p]) + y_end[p])
        for p in range(P):
            op = lambda v, qb_=qbar[p]: jfull(qb_, v)
            Qn[p * nsteps] = u0 + Dc[p]
            H = Dc[p]
            for k in range(1, nsteps):
                H = exp_action(op, plan_h, H)
                Qn[p * nsteps + k] += H
        Qn[S] = u0 + Dc[P]
        err = 0.0
        for p in range(P):
            a = Qn[p * nsteps:(p + 1) * nsteps + 1]
            b = Q[p * nsteps:(p + 1) * nsteps + 1]
            for m in range(B):
                num = float(np.sqrt(np.sum((a[:, m] - b[:, m]) ** 2)))
                den = float(np.sqrt(np.sum(b[:, m] ** 2)))
                err = max(err, num / den if den > 0 else num)
        history.append(err)
        Q = Qn
        if err < eps and it >= min_iter:
            return Q, it, history
    raise RuntimeError(f"no convergence after {max_iter} sweeps: {history}")


def burgers2d_nonlinear_tracking(nx, ny, D, T, P, nsteps, u0, f, law, target, plans_nl, plans_adj, eps,
                                 max_iter=25, min_iter=2):
    """The reference's loop with algorithm "nonlinear" (`optimization.py:206-231`): the iterative
    direct (Algorithm 2) for the trajectory, then `solve_adjoint_varying` with zero terminal data
    and the source 2(q − q_t) on the same equidistant partition — with q†_T = 0 the absorbed form
    is the hybrid's (zero-terminal slice solves + frozen spans), so the adjoint, cost and gradient
    are `burgers_tracking_hybrid`'s on the iterated trajectory."""
    Q, sweeps, history = burgers2d_iterative_direct(nx, ny, D, T, P, nsteps, u0, f, law, plans_nl, eps, max_iter,
                                                    min_iter)
    offs = np.arange(P + 1) * nsteps
    r = burgers_tracking_hybrid(nx, D, T, offs, u0, f, law, target, plans_adj, ny=ny, traj=Q)
    r.extras["sweeps"] = sweeps
    r.extras["history"] = history
    return r


# ---------------------------------------------------------------------------
# Equispaced checkpointing (`checkpointing.py:119-267`) over the config-mode pieces
# ---------------------------------------------------------------------------


def checkpointed_gradient(segment_gradient, direct_final, u0, M: int):
    """Rough forward sweep keeping M+1 segment-start states, then segments walked
    backward, each solved by ``segment_gradient(u_start, qdag_T)`` (``qdag_T`` None on
    the last segment: the objective's own terminal condition) and seeded with the
    carried q†. ``direct_final(u_start)`` is a segment's direct final state.
    Returns (J, grad, qdag0, G, uT, states)."""
    states = [np.asarray(u0, dtype=np.float64)]
    for _ in range(M):
        states.append(direct_final(states[-1]))
    grad = G = qd = J = uT = None
    for m in range(M, -1, -1):
        r = segment_gradient(states[m], qd)
        if qd is None:
            J, uT = r.J, r.uT
        grad = r.grad if grad is None else grad + r.grad
        G = r.G if G is None else G + r.G
        qd = r.qdag0
    return J, grad, qd, G, uT, states


# ---------------------------------------------------------------------------
# The reference's own hybrid loop (hybrid.py, optimization.py:172-189): tracking
# objective, forcing field × time law, Option B adjoint with an adjoint source,
# variable (geometric) slices — SURVEY §8(f) rank 2
# ---------------------------------------------------------------------------


def law_value(law, t):
    """θ(t) = α + β·sin(ωt) + γ·cos(ωt); the reference's forcing law is sin(ωt)
    (`problems.py:155-162`: α = γ = 0, β = 1)."""
    a, b, c, w = law
    return a + b * np.sin(w * t) + c * np.cos(w * t)


def law_substep_coef(plan: ChebPlan, law, t_top: float):
    """Series coefficients of ∫₀^τ θ(t_top − s)·e^{sM} ds (one substep of width τ, reflected
    time from t_top): α·τφ₁ + A·Gc + B·Gs with A = β sin ωt + γ cos ωt, B = −β cos ωt + γ sin ωt."""
    a, b, c, w = law
    if w == 0.0:
        return (a + c) * plan.coef_phi
    if plan.coef_gc is None or plan.omega != w:
        raise ValueError("plan lacks the time-law series for this ω")
    A = b * np.sin(w * t_top) + c * np.cos(w * t_top)
    Bc = -b * np.cos(w * t_top) + c * np.sin(w * t_top)
    return a * plan.coef_phi + A * plan.coef_gc + Bc * plan.coef_gs


def cheb_law_action(apply, plan: ChebPlan, v, G, law, t_top: float):
    """exp(span·M)v, and G += ∫₀^span θ(t_top − σ)·e^{σM}v dσ, by the plan's substeps."""
    c0, d, sigma = plan.center, plan.scale, float(plan.sigma)
    be = plan.coef_exp
    two_over = 2.0 / d
    tau = plan.span / plan.substeps
    y = v
    for j in range(plan.substeps):
        bl = law_substep_coef(plan, law, t_top - j * tau)
        u_prev = y
        acc = be[0] * u_prev
        lac = bl[0] * u_prev
        u_cur = (apply(u_prev) - c0 * u_prev) / d
        acc = acc + be[1] * u_cur
        lac = lac + bl[1] * u_cur
        for k in range(2, plan.degree + 1):
            u_next = two_over * (apply(u_cur) - c0 * u_cur) + sigma * u_prev
            u_prev, u_cur = u_cur, u_next
            acc = acc + be[k] * u_cur
            lac = lac + bl[k] * u_cur
        G += lac
        y = acc
    return y


def burgers_direct_law(u0, f, law, D, h_grid, h, S, rhs=None):
    """Serial classical RK4 of u' = −u∘Dx u + D·L u + θ(t)·f keeping every node (``rhs(u, f)``:
    another right-hand side, e.g. the 2D two-field one of `burgers_ops`)."""
    if rhs is not None:
        burgers_rhs = lambda u, ff, D_, h_: rhs(u, ff)  # noqa: E731 (shadows the 1D rhs below)
    else:
        burgers_rhs = globals()["burgers_rhs"]
    traj = np.empty((S + 1,) + u0.shape)
    u = u0.copy()
    traj[0] = u
    for i in range(S):
        t = i * h
        th1, th2, th4 = law_value(law, t), law_value(law, t + 0.5 * h), law_value(law, t + h)
        k1 = burgers_rhs(u, th1 * f, D, h_grid)
        k2 = burgers_rhs(u + (0.5 * h) * k1, th2 * f, D, h_grid)
        k3 = burgers_rhs(u + (0.5 * h) * k2, th2 * f, D, h_grid)
        k4 = burgers_rhs(u + h * k3, th4 * f, D, h_grid)
        u = u + (h / 6.0) * (k1 + 2.0 * k2 + 2.0 * k3 + k4)
        traj[i + 1] = u
    return traj


def slice_means_var(traj, offsets):
    """Trapezoid mean of each slice's nodes for variable slices (`problems.py:346-366`)."""
    out = []
    for p in range(len(offsets) - 1):
        a, b = int(offsets[p]), int(offsets[p + 1])
        w = np.ones(b - a + 1)
        w[0] = w[-1] = 0.5
        w /= (b - a)
        out.append(np.tensordot(w, traj[a:b + 1], axes=(0, 0)))
    return np.stack(out)


def tracking_cost(traj, target, T, h):
    """J = (1/T)·∫‖u − u_t‖² dt, trapezoid over the RK4 nodes (`optimization.py:84-93` on
    the node grid instead of a 200-point probe grid)."""
    d = traj - target
    e = np.sum(d * d, axis=-1)                 # (S+1, B)
    w = np.ones(e.shape[0])
    w[0] = w[-1] = 0.5
    return (h / T) * np.tensordot(w, e, axes=(0, 0))


def burgers_tracking_hybrid(nx, D, T, offsets, u0, f, law, target, plans_for, qdag_T=None, ny=None, traj=None):
    """The reference's hybrid loop with the configs' numerics.

    * direct: serial RK4 with forcing θ(t)·f (`hybrid.py:185-191`, `problems.py:155-162`);
    * cost: J = (1/T)∫‖u − u_t‖² dt (trapezoid on the nodes) — ``target`` (S+1, n) or (S+1, B, n);
    * adjoint, the reference's `solve_hybrid` (Option B, `hybrid.py:194-237`): per slice the
      inhomogeneous solve from zero terminal data with exact Jᵀ(u(t)) and the adjoint source
      s(t) = 2(u(t) − u_t(t)) (`optimization.py:96-100,172-175`), trajectory and target linearly
      interpolated at the stages; the slice ends are propagated through the frozen
      J(ū_m)ᵀ of every earlier slice (`propagate_span`, summed as one carry); a non-zero
      ``qdag_T`` adds the final span (`hybrid.py:232-233`);
    * gradient: ∂L/∂f = (1/T)∫ θ(t)·q†(t) dt (`optimization.py:103-112`), RK4-consistent in the
      slices and the planned series for the homogeneous parts.

    ``offsets``: the slices' node offsets (P+1 ints, 0 … S), h = T/S. ``plans_for(ubar)`` returns
    the per-slice plans (slice p of span (offsets[p+1]−offsets[p])·h). Returns an OracleResult
    whose ``grad`` is the field gradient (B, n). ``ny``: the reference's 2D two-field Burgers on
    an nx×ny grid (states, forcing, target and gradient of length 2·nx·ny, U block first)."""
    rhs2, adj2, n = burgers_ops(nx, D, ny)
    burgers_adjoint_apply = lambda u, y, D_, h_: adj2(u, y)  # noqa: E731 (1D or 2D operator)
    hg = 2.0 * np.pi / nx
    f = np.atleast_2d(np.asarray(f, dtype=np.float64))
    B = f.shape[0]
    u0 = np.broadcast_to(_as_batch(u0, n), (B, n)).copy()
    offsets = np.asarray(offsets, dtype=np.int64)
    P = len(offsets) - 1
    S = int(offsets[-1])
    h = T / S
    target = np.asarray(target, dtype=np.float64)
    tg = target[:, None, :] if target.ndim == 2 else target
    if traj is None:   # (a given direct trajectory: the nonlinear loop's, `optimization.py:206-225`)
        traj = burgers_direct_law(u0, f, law, D, hg, h, S, rhs=rhs2)
    J = tracking_cost(traj, tg, T, h)
    ubar = slice_means_var(traj, offsets)
    plans = plans_for(ubar)

    a_end = np.empty((P, B, n))
    zsum = np.zeros((B, n))
    for p in range(P):
        a = np.zeros((B, n))
        z = np.zeros((B, n))
        for i in range(int(offsets[p + 1] - offsets[p])):
            top = int(offsets[p + 1]) - i
            ua, ub = traj[top], traj[top - 1]
            um = 0.5 * ua + 0.5 * ub
            ta, tb = tg[top], tg[top - 1]
            tm = 0.5 * ta + 0.5 * tb
            sa, sm, sb = 2.0 * (ua - ta), 2.0 * (um - tm), 2.0 * (ub - tb)
            t_a = top * h
            th_a, th_m, th_b = law_value(law, t_a), law_value(law, t_a - 0.5 * h), law_value(law, t_a - h)
            k1 = burgers_adjoint_apply(ua, a, D, hg) + sa
            Y2 = a + (0.5 * h) * k1
            k2 = burgers_adjoint_apply(um, Y2, D, hg) + sm
            Y3 = a + (0.5 * h) * k2
            k3 = burgers_adjoint_apply(um, Y3, D, hg) + sm
            Y4 = a + h * k3
            k4 = burgers_adjoint_apply(ub, Y4, D, hg) + sb
            z = z + (h / 6.0) * (th_a * a + 2.0 * th_m * (Y2 + Y3) + th_b * Y4)
            a = a + (h / 6.0) * (k1 + 2.0 * k2 + 2.0 * k3 + k4)
        a_end[p] = a
        zsum += z

    Gh = np.zeros((B, n))
    if qdag_T is not None:
        C = np.broadcast_to(_as_batch(qdag_T, n), (B, n)).copy()
        top_p = P - 1
    else:
        C = a_end[P - 1].copy()
        top_p = P - 2
    for p in range(top_p, -1, -1):
        ub_ = ubar[p]
        C = cheb_law_action(lambda y, ub_=ub_: burgers_adjoint_apply(ub_, y, D, hg), plans[p], C, Gh, law,
                            float(offsets[p + 1]) * h)
        if not (qdag_T is None and p == P - 1):
            C = C + a_end[p]
    grad = (zsum + Gh) / T
    return OracleResult(J=J, grad=grad, uT=traj[-1], qdag0=C, G=grad,
                        extras={"traj": traj, "ubar": ubar, "plans": plans, "a_end": a_end, "zsum": zsum,
                                "Gh": Gh})


# ---------------------------------------------------------------------------
# Linear testbed with a forcing time law θ(t) (the reference's f·sin(ωt),
# `problems.py:155-162`) and the terminal objective
# ---------------------------------------------------------------------------


def rk4_linear_law(apply, g0, f, law, t0: float, h: float, nsteps: int):
    """Zero-data classical RK4 for y' = M y + g0 + θ(t)·f from t0 (θ at the stage times)."""
    y = np.zeros_like(f)
    for k in range(nsteps):
        t = t0 + k * h
        th1, th2, th4 = law_value(law, t), law_value(law, t + 0.5 * h), law_value(law, t + h)
        k1 = apply(y) + g0 + th1 * f
        k2 = apply(y + (0.5 * h) * k1) + g0 + th2 * f
        k3 = apply(y + (0.5 * h) * k2) + g0 + th2 * f
        k4 = apply(y + h * k3) + g0 + th4 * f
        y = y + (h / 6.0) * (k1 + 2.0 * k2 + 2.0 * k3 + k4)
    return y


def rk4_adjoint_law(apply, c, law, t_top: float, h: float, nsteps: int):
    """Zero-data RK4 in reflected time of w' = M w + c from t_top down, with the θ-weighted
    RK4-consistent integral z = ∫θ(t)·w dt (RK4 on (w, z)' = (M w + c, θ(t_top − σ)·w))."""
    w = np.zeros_like(c)
    z = np.zeros_like(c)
    for k in range(nsteps):
        t = t_top - k * h
        ta, tm, tb = law_value(law, t), law_value(law, t - 0.5 * h), law_value(law, t - h)
        k1 = apply(w) + c
        Y2 = w + (0.5 * h) * k1
        k2 = apply(Y2) + c
        Y3 = w + (0.5 * h) * k2
        k3 = apply(Y3) + c
        Y4 = w + h * k3
        k4 = apply(Y4) + c
        z = z + (h / 6.0) * (ta * w + 2.0 * tm * (Y2 + Y3) + tb * Y4)
        w = w + (h / 6.0) * (k1 + 2.0 * k2 + 2.0 * k3 + k4)
    return w, z


def law_integral(law, T: float) -> float:
    """∫₀ᵀ θ(t) dt."""
    a, b, c, w = law
    if w == 0.0:
        return (a + c) * T
    return a * T + b * (1.0 - np.cos(w * T)) / w + c * np.sin(w * T) / w


def linear_gradient_law(grid_nx, grid_ny, A, basis, T, P, nsteps, u0, u_target, ctrl, law, plan_slice):
    """One Paraexp direct-adjoint gradient of the linear testbed with the forcing f·θ(t) and the
    terminal objective (single-rank scan). Every slice solves its own RK4 problem (θ shifts with
    T_p); the carry is unchanged; the adjoint's ∂J/∂f = ∫θ(t)·q†(t) dt gathers the θ-weighted
    lane integrals, ∫θ dt·q†_T and the law series of every carry (`law_substep_coef`)."""
    nx, ny = grid_nx, grid_ny
    n = nx * ny
    ctrl = np.atleast_2d(np.asarray(ctrl, dtype=np.float64))
    B = ctrl.shape[0]
    u0 = np.broadcast_to(_as_batch(u0, n), (B, n))
    ut = np.broadcast_to(_as_batch(u_target, n), (B, n))
    AT = tuple(np.asarray(A)[[0, 2, 1, 4, 3]])
    applyA = lambda u: stencil_apply(A, u, nx, ny)
    applyAT = lambda u: stencil_apply(AT, u, nx, ny)
    delta = T / P
    h = delta / nsteps
    f = basis.field(ctrl)
    g0 = applyA(u0)
    D = None
    for p in range(P):
        v = rk4_linear_law(applyA, g0, f, law, p * delta, h, nsteps)
        D = v if p == 0 else exp_action(applyA, plan_slice, D) + v
    uT = u0 + D
    qT = uT - ut
    J = 0.5 * np.sum(qT * qT, axis=1)
    c = applyAT(qT)
    C = None
    G = law_integral(law, T) * qT
    for p in range(P - 1, -1, -1):
        w, z = rk4_adjoint_law(applyAT, c, law, (p + 1) * delta, h, nsteps)
        G = G + z
        if p == P - 1:
            C = w
        else:
            C = cheb_law_action(applyAT, plan_slice, C, G, law, (p + 1) * delta) + w
    qdag0 = qT + C
    grad = basis.project(G)
    return OracleResult(J=J, grad=grad, uT=uT, qdag0=qdag0, G=G)


# ---------------------------------------------------------------------------
# The reference's linear loop with its own objective (`optimization.py:154-231`, algorithm
# "linear"): Paraexp direct with the forcing f·θ(t), tracking cost, adjoint with the source
# 2(q − q_true) and zero terminal data, ∂L/∂f = (1/T)∫θ·q† dt
# ---------------------------------------------------------------------------


def rk4_full_law(apply, y0, f, law, t0: float, h: float, nsteps: int):
    """Classical RK4 of y' = M y + θ(t)·f from y0, every node kept: (nsteps+1, B, n)."""
    out = np.empty((nsteps + 1,) + y0.shape)
    y = y0.copy()
    out[0] = y
    for k in range(nsteps):
        t = t0 + k * h
        th1, th2, th4 = law_value(law, t), law_value(law, t + 0.5 * h), law_value(law, t + h)
        k1 = apply(y) + th1 * f
        k2 = apply(y + (0.5 * h) * k1) + th2 * f
        k3 = apply(y + (0.5 * h) * k2) + th2 * f
        k4 = apply(y + h * k3) + th4 * f
        y = y + (h / 6.0) * (k1 + 2.0 * k2 + 2.0 * k3 + k4)
        out[k + 1] = y
    return out


def linear_tracking_gradient(grid_nx, grid_ny, A, basis, T, P, nsteps, u0, ctrl, law, target, plan_slice):
    """Config-mode restatement of the reference's linear loop (single-rank scan):

    * direct: the Paraexp direct of `linear_gradient_law` gives the slice-edge states u(T_p)
      (absorbed u0, every slice's own RK4 lane, summed-chain carries); the solution inside slice p
      is the RK4 sweep of u' = A u + θ(t) f from u(T_p) over the slice's steps (by linearity the
      lane plus the homogeneous propagation of the incoming state, `paraexp.py:202-218`);
    * cost J = (1/T)∫‖u − u_t‖² dt, trapezoid on the RK4 nodes;
    * adjoint (`solve_adjoint_linear` with adj_forcing = 2(q − q_true), zero terminal data,
      `paraexp.py:298-326`): per slice a' = Aᵀa + 2(u − u_t) from a = 0 at T_{p+1} in reflected time
      (trajectory and target linearly interpolated at the half steps), the θ-weighted
      RK4-consistent ∫; the slice ends carried through exp(ΔAᵀ) with the law series;
    * ∂L/∂f = (1/T)(Σ z_p + Σ carry integrals) (`gradient_wrt_forcing`), on the basis (field or modes).
    Returns an OracleResult (grad projected on the basis; G the field gradient)."""
    nx, ny = grid_nx, grid_ny
    n = nx * ny
    ctrl = np.atleast_2d(np.asarray(ctrl, dtype=np.float64))
    B = ctrl.shape[0]
    u0 = np.broadcast_to(_as_batch(u0, n), (B, n)).copy()
    AT = tuple(np.asarray(A)[[0, 2, 1, 4, 3]])
    applyA = lambda u: stencil_apply(A, u, nx, ny)
    applyAT = lambda u: stencil_apply(AT, u, nx, ny)
    delta = T / P
    h = delta / nsteps
    S = P * nsteps
    f = basis.field(ctrl)
    g0 = applyA(u0)
    # slice-edge states by the Paraexp direct (the same operation sequence as linear_gradient_law)
    edges = [u0.copy()]
    D = None
    for p in range(P):
        v = rk4_linear_law(applyA, g0, f, law, p * delta, h, nsteps)
        D = v if p == 0 else exp_action(applyA, plan_slice, D) + v
        edges.append(u0 + D)
    # the trajectory inside every slice from its edge state
    traj = np.empty((S + 1, B, n))
    traj[0] = u0
    for p in range(P):
        seg = rk4_full_law(applyA, edges[p], f, law, p * delta, h, nsteps)
        traj[p * nsteps + 1:(p + 1) * nsteps + 1] = seg[1:]
    tg = np.asarray(target, dtype=np.float64)
    tg = tg[:, None, :] if tg.ndim == 2 else tg
    J = tracking_cost(traj, tg, T, h)
    a_end = np.empty((P, B, n))
    zsum = np.zeros((B, n))
    for p in range(P):
        a = np.zeros((B, n))
        z = np.zeros((B, n))
        for i in range(nsteps):
            top = (p + 1) * nsteps - i
            ua, ub = traj[top], traj[top - 1]
            ta, tb = tg[top], tg[top - 1]
            sa, sb = 2.0 * (ua - ta), 2.0 * (ub - tb)
            sm = 2.0 * ((0.5 * ua + 0.5 * ub) - (0.5 * ta + 0.5 * tb))
            t_a = top * h
            th_a, th_m, th_b = law_value(law, t_a), law_value(law, t_a - 0.5 * h), law_value(law, t_a - h)
            k1 = applyAT(a) + sa
            Y2 = a + (0.5 * h) * k1
            k2 = applyAT(Y2) + sm
            Y3 = a + (0.5 * h) * k2
            k3 = applyAT(Y3) + sm
            Y4 = a + h * k3
            k4 = applyAT(Y4) + sb
            z = z + (h / 6.0) * (th_a * a + 2.0 * th_m * (Y2 + Y3) + th_b * Y4)
            a = a + (h / 6.0) * (k1 + 2.0 * k2 + 2.0 * k3 + k4)
        a_end[p] = a
        zsum += z
    C = a_end[P - 1].copy()
    Gh = np.zeros((B, n))
    for p in range(P - 2, -1, -1):
        C = cheb_law_action(applyAT, plan_slice, C, Gh, law, (p + 1) * delta) + a_end[p]
    G = (zsum + Gh) / T
    # u(T) is the Paraexp direct's (the last edge state), as the reference's direct.eval(T); the
    # recorded node S differs from it by the RK4 error of the homogeneous propagation over slice P−1
    return OracleResult(J=J, grad=basis.project(G), uT=edges[-1], qdag0=C, G=G,
                        extras={"traj": traj, "edges": np.stack(edges), "a_end": a_end})
