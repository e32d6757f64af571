"""A-priori planning of the Chebyshev / Krylov exponential actions.

The reference propagates homogeneous problems with the real-Leja-point method
(`pkg/src/paradjoint/timestepping.py:306-423`): degree and substeps are found
*adaptively* from a Newton-correction test, on a Gershgorin interval of the
real axis (`timestepping.py:260-266`). BASELINE configs ask for Chebyshev
(tol 1e-12 / 1e-10) and Krylov (m=30, tol 1e-10) actions instead, and the
GPU/CPU parity bar needs both sides to execute the *same* operation sequence.
So everything data-dependent is decided here, once, on the host:

* the spectrum enclosure is exact for the circulant advection–diffusion
  operator (a Minkowski sum of ellipses, see ``problems.advdiff_region``) —
  unlike the real Gershgorin interval, it stays valid for advection-dominated
  spectra (cell Péclet > 2, where the reference's interval has a positive
  upper end and its Newton test is fooled);
* Chebyshev polynomials are taken on the focal segment of an ellipse (real
  foci c0 ± d, or imaginary foci c0 ± i·d); with imaginary foci the
  recurrence ``U_{k+1} = 2·X·U_k + U_{k-1}`` stays real (σ = +1), with real foci
  it is the classical ``U_{k+1} = 2·X·U_k − U_{k-1}`` (σ = −1), X = (M−c0)/d;
* degree and substep count are the cheapest pair whose truncation error, evaluated
  on the boundary of the enclosure (max-modulus principle), is below the
  tolerance, and whose rounding amplification is bounded.

The exp and φ₁ coefficient sets share one basis recurrence: the adjoint sweep
needs ∫ q† dt, i.e. τ·φ₁(τB)·C alongside exp(τB)·C.
"""

from __future__ import annotations

from dataclasses import dataclass, field, replace
import math
from functools import lru_cache

import numpy as np

from .errors import PropagationFailure
from .problems import SpectralRegion

EPS = 2.220446049250313e-16


@dataclass(frozen=True)
class ChebyshevConfig:
    """Chebyshev exp-action settings (BASELINE configs 1, 2, 3, 5)."""

    tol: float = 1e-12
    max_degree: int = 120
    substep_limit: int = 1 << 16
    # 0: ``tol`` bounds each action. > 0: ``tol`` is the error budget of the composite
    # propagation over this horizon (the P sequential slice carries of a sweep): an action of
    # span τ is planned to tol·(τ/horizon)/HORIZON_MARGIN, so the scan and every block-scan
    # decomposition of it agree to well below ``tol`` (SURVEY §8(e) G-invariance)
    horizon: float = 0.0

    def __post_init__(self):
        if self.tol <= 0:
            raise ValueError("tol must be positive")
        if self.max_degree < 2:
            raise ValueError("max_degree must be at least 2")
        if self.horizon < 0:
            raise ValueError("horizon must be non-negative")


@dataclass(frozen=True)
class KrylovConfig:
    """Arnoldi exp-action settings (BASELINE config 4: m = 30, tol 1e-10)."""

    m: int = 30
    tol: float = 1e-10
    substep_limit: int = 1 << 16
    horizon: float = 0.0  # as ChebyshevConfig.horizon

    def __post_init__(self):
        if self.m < 2:
            raise ValueError("need at least 2 Krylov vectors")
        if self.tol <= 0:
            raise ValueError("tol must be positive")
        if self.horizon < 0:
            raise ValueError("horizon must be non-negative")


@dataclass(frozen=True)
class ChebPlan:
    """One span τ = substeps·τ_s; per substep out = Σ_k coef_exp[k]·U_k,
    phi_out += Σ_k coef_phi[k]·U_k (= τ_s·φ₁(τ_s M)·y)."""

    span: float
    substeps: int
    degree: int
    center: float
    scale: float
    sigma: int
    coef_exp: np.ndarray = field(repr=False)
    coef_phi: np.ndarray = field(repr=False)
    err_bound: float = 0.0
    # time-law integrals (``omega`` > 0, the hybrid tracking path): per substep of width τ_s,
    # Σ_k coef_gc[k]·U_k = ∫₀^τ_s cos(ωs)·e^{sM} ds·y and Σ_k coef_gs[k]·U_k = ∫₀^τ_s sin(ωs)·e^{sM} ds·y
    omega: float = 0.0
    coef_gc: np.ndarray | None = field(default=None, repr=False)
    coef_gs: np.ndarray | None = field(default=None, repr=False)

    @property
    def terms(self) -> int:
        """Operator applications per action (the unit the roofline counts)."""
        return self.substeps * self.degree


@dataclass(frozen=True)
class KrylovPlan:
    span: float
    substeps: int
    m: int

    @property
    def terms(self) -> int:
        return self.substeps * self.m


def phi1(z: np.ndarray) -> np.ndarray:
    """φ₁(z) = (e^z − 1)/z, stable near 0 (complex-safe)."""
    z = np.asarray(z, dtype=np.complex128)
    out = np.empty_like(z)
    small = np.abs(z) < 0.5
    zs = z[small]
    acc = np.zeros_like(zs)
    term = np.ones_like(zs)
    for j in range(1, 24):
        acc += term
        term = term * zs / (j + 1)
    out[small] = acc
    zb = z[~small]
    # e^z − 1 = (e^x·cos y − 1) + i·e^x·sin y; expm1 keeps the real part accurate
    out[~small] = (np.expm1(zb.real) + np.exp(zb.real) * (np.cos(zb.imag) - 1.0)
                   + 1j * np.exp(zb.real) * np.sin(zb.imag)) / zb
    return out


def law_integrals(z: np.ndarray, tau: float, omega: float) -> tuple[np.ndarray, np.ndarray]:
    """(Gc, Gs)(z) = ∫₀^τ (cos ωs, sin ωs)·e^{sz} ds, from τφ₁(τ(z ± iω)) (complex-safe)."""
    z = np.asarray(z, dtype=np.complex128)
    ep = tau * phi1(tau * (z + 1j * omega))
    em = tau * phi1(tau * (z - 1j * omega))
    return 0.5 * (ep + em), (ep - em) / 2j


def chebyshev_coefficients(f, center: float, d: float, imag: bool, n: int) -> np.ndarray:
    """Real recurrence coefficients b_k of f on the focal segment.

    a_k are the Chebyshev coefficients of w ↦ f(c0 + d·w) (real foci) or
    f(c0 + i·d·w) (imaginary foci) on [−1, 1], from a DCT at n Chebyshev
    points; for imaginary foci b_k = a_k·(−i)^k (real because
    f(c0 − i·d·w) = conj f(c0 + i·d·w)).
    """
    j = np.arange(n)
    theta = np.pi * (j + 0.5) / n
    w = np.cos(theta)
    z = center + (1j * d * w if imag else d * w)
    F = f(z)
    k = np.arange(n)[:, None]
    a = (2.0 / n) * (np.cos(k * theta[None, :]) @ F)
    a[0] *= 0.5
    if imag:
        a = a * (-1j) ** np.arange(n)
    return np.real(a)


def _evaluate(region_pts: np.ndarray, crouzeix: float, center: float, d: float,
              imag: bool, tau: float, kmax: int):
    """Truncation errors (exp, φ₁) and rounding estimates for degrees 0..kmax.

    Candidates whose coefficients overflow yield non-finite errors and are
    rejected by the caller's comparisons.
    """
    with np.errstate(all="ignore"):
        return _evaluate_impl(region_pts, crouzeix, center, d, imag, tau, kmax)


def _evaluate_impl(region_pts, crouzeix, center, d, imag, tau, kmax):
    nq = max(64, 2 * kmax + 32)
    be = chebyshev_coefficients(lambda z: np.exp(tau * z), center, d, imag, nq)[: kmax + 1]
    bp = chebyshev_coefficients(lambda z: tau * phi1(tau * z), center, d, imag, nq)[: kmax + 1]
    sigma = 1.0 if imag else -1.0
    X = (region_pts - center) / d
    fe = np.exp(tau * region_pts)
    fp = tau * phi1(tau * region_pts)
    U0 = np.ones_like(X)
    U1 = X.copy()
    Se = be[0] * U0
    Sp = bp[0] * U0
    err_e = np.empty(kmax + 1)
    err_p = np.empty(kmax + 1)
    rnd = np.empty(kmax + 1)
    err_e[0] = np.max(np.abs(Se - fe))
    err_p[0] = np.max(np.abs(Sp - fp))
    acc_r = abs(be[0]) + abs(bp[0]) / max(tau, 1e-300)
    rnd[0] = acc_r
    Uprev, Ucur = U0, U1
    for k in range(1, kmax + 1):
        if k > 1:
            Unext = 2.0 * X * Ucur + sigma * Uprev
            Uprev, Ucur = Ucur, Unext
        g = np.max(np.abs(Ucur))
        Se = Se + be[k] * Ucur
        Sp = Sp + bp[k] * Ucur
        err_e[k] = np.max(np.abs(Se - fe))
        err_p[k] = np.max(np.abs(Sp - fp))
        acc_r += (abs(be[k]) + abs(bp[k]) / max(tau, 1e-300)) * g
        rnd[k] = acc_r
    return (crouzeix * err_e, crouzeix * err_p / max(tau, 1e-300),
            2.0 * EPS * crouzeix * rnd, be, bp)


def _first_feasible(pts, crouzeix, center, d, imag, tau, kmax, tol_s, with_rounding, kcap, omega=0.0):
    """Smallest degree K (≥ 1) whose exp and φ₁ truncation errors (and rounding
    estimate) meet tol_s at K and K+1 — the same arithmetic as `_evaluate`, but
    stopping as soon as K is found, the monotone rounding estimate exceeds its
    budget, or K could no longer beat the best plan so far (``kcap``)."""
    with np.errstate(all="ignore"):
        nq = max(64, 2 * kmax + 32)
        be = chebyshev_coefficients(lambda z: np.exp(tau * z), center, d, imag, nq)[: kmax + 1]
        bp = chebyshev_coefficients(lambda z: tau * phi1(tau * z), center, d, imag, nq)[: kmax + 1]
        # the time-law integral series (omega > 0) are held to the φ₁ series' bound
        law = []
        if omega > 0.0:
            for j in range(2):
                fl = lambda z, j=j: law_integrals(z, tau, omega)[j]
                law.append((chebyshev_coefficients(fl, center, d, imag, nq)[: kmax + 1], fl(pts)))
        if not (np.all(np.isfinite(be)) and np.all(np.isfinite(bp))
                and all(np.all(np.isfinite(c)) for c, _ in law)):
            return None
        sigma = 1.0 if imag else -1.0
        X = (pts - center) / d
        fe = np.exp(tau * pts)
        fp = tau * phi1(tau * pts)
        ptau = max(tau, 1e-300)
        Uprev, Ucur = np.ones_like(X), X.copy()
        Se = be[0] * Uprev
        Sp = bp[0] * Uprev
        Sl = [c[0] * Uprev for c, _ in law]
        acc_r = abs(be[0]) + abs(bp[0]) / ptau + sum(abs(c[0]) for c, _ in law) / ptau
        prev_ok = False
        errs = []
        for k in range(0, kmax + 1):
            if k >= 1:
                if k > 1:
                    Unext = 2.0 * X * Ucur + sigma * Uprev
                    Uprev, Ucur = Ucur, Unext
                g = np.max(np.abs(Ucur))
                Se = Se + be[k] * Ucur
                Sp = Sp + bp[k] * Ucur
                for j, (c, _) in enumerate(law):
                    Sl[j] = Sl[j] + c[k] * Ucur
                acc_r += (abs(be[k]) + abs(bp[k]) / ptau + sum(abs(c[k]) for c, _ in law) / ptau) * g
            ee = crouzeix * np.max(np.abs(Se - fe))
            ep = crouzeix * np.max(np.abs(Sp - fp)) / ptau
            for j, (_, fv) in enumerate(law):
                ep = max(ep, crouzeix * np.max(np.abs(Sl[j] - fv)) / ptau)
            rr = 2.0 * EPS * crouzeix * acc_r
            errs.append(max(ee, ep))
            if with_rounding and not rr <= 0.5 * tol_s:
                return None
            ok = ee <= tol_s and ep <= tol_s
            if ok and prev_ok:
                K = max(k - 1, 1)
                extra = tuple(c[: K + 1].copy() for c, _ in law)
                return K, be[: K + 1].copy(), bp[: K + 1].copy(), float(errs[K]), extra
            prev_ok = ok
            if kcap is not None and k - 1 > kcap:
                return None
    return None


def _foci_candidates(region: SpectralRegion):
    lo, hi, im = region.box()
    c0 = 0.5 * (lo + hi)
    alpha = 0.5 * (hi - lo)
    beta = im
    cands = []
    for kappa in (0.5, 0.75, 1.0, 1.25, 1.5, 2.0, 3.0):
        if beta > 0:
            cands.append((c0, kappa * beta, True))
        if alpha > 0:
            cands.append((c0, kappa * alpha, False))
    if not cands:
        cands.append((c0, 1.0, False))
    return cands


_SUBSTEPS = (1, 2, 3, 4, 5, 6, 8, 10, 12, 16, 20, 24, 32, 40, 48, 64, 80, 96, 128,
             160, 192, 256, 320, 384, 512, 640, 768, 1024, 1536, 2048, 3072, 4096,
             6144, 8192, 12288, 16384, 24576, 32768, 49152, 65536)


def _plan_cheb(region: SpectralRegion, span: float, tol: float, max_degree: int,
               substep_limit: int, with_rounding: bool = True, omega: float = 0.0) -> ChebPlan:
    pts = region.boundary(1024)
    best = None
    for (c0, d, imag) in _foci_candidates(region):
        for s in _SUBSTEPS:
            if s > substep_limit:
                break
            if best is not None and s * 2 >= best[0]:
                break
            tau = span / s
            tol_s = tol / s
            # degree bound beyond which this (foci, s) cannot beat the best plan so far
            kcap = None if best is None else best[0] // s
            # the next degree must satisfy the bound too (no lucky dip)
            found = _first_feasible(pts, region.crouzeix, c0, d, imag, tau, max_degree, tol_s,
                                    with_rounding, kcap, omega)
            if found is None:
                continue
            K, be, bp, err, extra = found
            cost = s * K
            if best is None or cost < best[0]:
                best = (cost, c0, d, imag, s, K, be, bp, err, extra)
    if best is None:
        raise PropagationFailure(
            f"no Chebyshev plan within {substep_limit} substeps of degree <= {max_degree} "
            f"reaches tol={tol:g} over span {span:g}")
    _, c0, d, imag, s, K, be, bp, err, extra = best
    gc, gs = extra if extra else (None, None)
    return ChebPlan(span=span, substeps=s, degree=K, center=c0, scale=d,
                    sigma=1 if imag else -1, coef_exp=be, coef_phi=bp, err_bound=err,
                    omega=float(omega), coef_gc=gc, coef_gs=gs)


def _region_key(region: SpectralRegion):
    return (region.ellipses, region.rect, region.crouzeix)


@lru_cache(maxsize=256)
def _plan_cached(key, span, tol, max_degree, substep_limit, omega=0.0):
    ellipses, rect, crouzeix = key
    region = SpectralRegion(ellipses=ellipses, rect=rect, crouzeix=crouzeix)
    return _plan_cheb(region, span, tol, max_degree, substep_limit, omega=omega)


def plan_chebyshev(region: SpectralRegion, span: float, cfg: ChebyshevConfig, omega: float = 0.0) -> ChebPlan:
    """Cheapest (foci, substeps, degree) reaching ``cfg.tol`` over ``span``; with ``omega`` > 0
    the plan also carries the time-law integral series (``coef_gc``, ``coef_gs``), held to
    the same bound."""
    if span <= 0:
        raise ValueError("span must be positive")
    if omega < 0:
        raise ValueError("omega must be non-negative")
    return _plan_cached(_region_key(region), float(span), float(cfg.tol),
                        int(cfg.max_degree), int(cfg.substep_limit), float(omega))


@lru_cache(maxsize=64)
def _krylov_cached(key, span, m, tol, substep_limit):
    ellipses, rect, crouzeix = key
    region = SpectralRegion(ellipses=ellipses, rect=rect, crouzeix=crouzeix)
    pts = region.boundary(1024)
    # Arnoldi error <= 2·min_{p in P_{m-1}} max_{W(A)} |e^{τλ} − p(λ)| (normal A):
    # take the smallest substep count at which some degree-(m−1) Chebyshev
    # partial sum already meets tol/2 on the enclosure.
    for s in _SUBSTEPS:
        if s > substep_limit:
            break
        tau = span / s
        for (c0, d, imag) in _foci_candidates(region):
            ee, ep, _, _, _ = _evaluate(pts, region.crouzeix, c0, d, imag, tau, m - 1)
            if ee[m - 1] <= 0.5 * tol / s and ep[m - 1] <= 0.5 * tol / s:
                return KrylovPlan(span=span, substeps=s, m=m)
    raise PropagationFailure(f"no Krylov substep count within {substep_limit} reaches tol={tol:g}")


def plan_krylov(region: SpectralRegion, span: float, cfg: KrylovConfig) -> KrylovPlan:
    if span <= 0:
        raise ValueError("span must be positive")
    return _krylov_cached(_region_key(region), float(span), int(cfg.m), float(cfg.tol),
                          int(cfg.substep_limit))


def chained(plan, k: int):
    """The same per-substep series applied k times in a row: span k·τ (always
    feasible; accuracy that of k consecutive base actions, i.e. of the scan)."""
    if isinstance(plan, KrylovPlan):
        return KrylovPlan(span=plan.span * k, substeps=plan.substeps * k, m=plan.m)
    return ChebPlan(span=plan.span * k, substeps=plan.substeps * k, degree=plan.degree, center=plan.center,
                    scale=plan.scale, sigma=plan.sigma, coef_exp=plan.coef_exp, coef_phi=plan.coef_phi,
                    err_bound=plan.err_bound * k, omega=plan.omega, coef_gc=plan.coef_gc, coef_gs=plan.coef_gs)


HORIZON_MARGIN = 10.0


def action_config(cfg, span: float):
    """The per-action settings for an action of ``span``: ``cfg`` itself, or with a
    horizon budget (``cfg.horizon`` > 0) the tolerance tol·(span/horizon)/HORIZON_MARGIN."""
    if cfg.horizon <= 0:
        return cfg
    return replace(cfg, tol=cfg.tol * min(1.0, span / cfg.horizon) / HORIZON_MARGIN, horizon=0.0)


def plan_for(region: SpectralRegion, span: float, cfg, base_span: float | None = None, omega: float = 0.0):
    """Plan for ``span``; when ``span`` is an integer multiple k of ``base_span``
    (block-scan long spans are multiples of the slice width), the k-fold chained
    base plan is also considered and the cheaper feasible plan is returned. A horizon
    budget (``cfg.horizon``) is split over the actions in proportion to their spans."""
    if isinstance(cfg, KrylovConfig):
        if omega:
            raise PropagationFailure("a forcing time law needs Chebyshev exp-actions (its integral series)")
        one = lambda reg, sp, c: plan_krylov(reg, sp, action_config(c, sp))
    else:
        one = lambda reg, sp, c: plan_chebyshev(reg, sp, action_config(c, sp), omega)
    k = None
    if base_span is not None and span > base_span:
        q = span / base_span
        if abs(q - round(q)) <= 1e-9 * q:
            k = int(round(q))
    if k is None:
        return one(region, span, cfg)
    base = chained(one(region, base_span, cfg), k)
    try:
        direct = one(region, span, cfg)
    except PropagationFailure:
        return base
    return direct if direct.terms <= base.terms else base


def plan_family(region: SpectralRegion, spans, cfg: ChebyshevConfig, omega: float = 0.0) -> list[ChebPlan]:
    """Cached `_plan_family` (the frozen-operator regions are quantised, so repeated loops on
    the same problem reuse the plans)."""
    spans = tuple(float(s) for s in spans)
    return list(_plan_family_cached(_region_key(region), spans, cfg, float(omega)))


@lru_cache(maxsize=64)
def _plan_family_cached(key, spans, cfg, omega):
    ellipses, rect, crouzeix = key
    return tuple(_plan_family(SpectralRegion(ellipses=ellipses, rect=rect, crouzeix=crouzeix), spans, cfg, omega))


def _plan_family(region: SpectralRegion, spans, cfg: ChebyshevConfig, omega: float = 0.0) -> list[ChebPlan]:
    """Plans for a set of slice spans sharing one spectral region (variable slices, e.g. the
    hybrid's geometric partition): the widest span is planned in full; every other span reuses
    its foci with as many substeps as keep the substep width at most the widest plan's, and the
    smallest degree that meets the same bounds at its own
    substep width (a DCT and one series evaluation instead of a full search), falling back to
    a full plan if none does."""
    spans = [float(s) for s in spans]
    if not spans or min(spans) <= 0:
        raise ValueError("spans must be positive")
    cfg1 = action_config(cfg, max(spans))
    base = plan_chebyshev(region, max(spans), cfg1, omega)
    pts = region.boundary(1024)
    out: dict[float, ChebPlan] = {max(spans): base}
    for sp in sorted(set(spans)):
        if sp in out:
            continue
        c = action_config(cfg, sp)
        s = max(1, math.ceil(base.substeps * sp / base.span - 1e-9))  # substep width ≤ the base's
        found = _first_feasible(pts, region.crouzeix, base.center, base.scale, base.sigma > 0, sp / s,
                                base.degree + 8, c.tol / s, True, None, omega)
        if found is None:
            out[sp] = plan_chebyshev(region, sp, c, omega)
            continue
        K, be, bp, err, extra = found
        gc, gs = extra if extra else (None, None)
        out[sp] = ChebPlan(span=sp, substeps=s, degree=K, center=base.center, scale=base.scale,
                           sigma=base.sigma, coef_exp=be, coef_phi=bp, err_bound=err, omega=float(omega),
                           coef_gc=gc, coef_gs=gs)
    return [out[s] for s in spans]
