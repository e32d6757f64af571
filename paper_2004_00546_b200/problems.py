"""Periodic stencil problems of the Paraexp path (host-side description).

Restates, for the BASELINE configs, the testbeds of the reference's
`pkg/src/paradjoint/problems.py`:

* grids are periodic on [0, 2π) (1D) or [0, 2π)² (2D) with x fastest in the
  flat index ``i + nx*j`` (`problems.py:25-56`);
* the linear operator is second-order central differences,
  A = −a_x·∂x − a_y·∂y + D·∇² (`problems.py:106-152`), with per-axis advection
  (the reference has one scalar ``a``; BASELINE configs 4–5 need a=(1, 0.5));
* Burgers is the reference's system with V ≡ 0 (`problems.py:177-194`,
  `:316-343`), i.e. the 1D viscous Burgers equation in U.

Nothing here computes on the GPU: it produces the stencil coefficients, the
Fourier control basis and the spectral enclosures that the native sweeps and
the exponential-action planner consume.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

TWO_PI = 2.0 * np.pi

ADVECTION_DIFFUSION = "advection_diffusion"
BURGERS = "burgers"


@dataclass(frozen=True)
class Grid:
    """Uniform periodic grid: 1D when ``ny == 1``, else 2D (`problems.py:25-56`)."""

    nx: int
    ny: int = 1

    def __post_init__(self):
        if self.nx < 3:
            raise ValueError("grid needs nx >= 3 for the periodic stencil")
        if self.ny != 1 and self.ny < 3:
            raise ValueError("2D grid needs ny >= 3 for the periodic stencil")

    @property
    def dim(self) -> int:
        return 1 if self.ny == 1 else 2

    @property
    def hx(self) -> float:
        return TWO_PI / self.nx

    @property
    def hy(self) -> float:
        return TWO_PI / self.ny if self.ny > 1 else 1.0

    @property
    def npoints(self) -> int:
        return self.nx * self.ny

    def x1(self) -> np.ndarray:
        return np.arange(self.nx) * self.hx

    def y1(self) -> np.ndarray:
        return np.arange(self.ny) * self.hy if self.ny > 1 else np.zeros(1)

    def coordinates(self) -> tuple[np.ndarray, np.ndarray]:
        """Flat x and y coordinate arrays in the state layout (`problems.py:51-56`)."""
        xg, yg = np.meshgrid(self.x1(), self.y1(), indexing="xy")
        return xg.ravel(), yg.ravel()


@dataclass(frozen=True)
class ProblemSpec:
    """Equation kind and coefficients (`problems.py:59-83`, per-axis ``a``)."""

    kind: str
    a: tuple[float, float]
    D: float
    T: float

    def __post_init__(self):
        if self.kind not in (ADVECTION_DIFFUSION, BURGERS):
            raise ValueError(f"unknown problem kind {self.kind!r}")
        if self.D <= 0:
            raise ValueError("diffusion coefficient D must be positive")
        if self.T <= 0:
            raise ValueError("final time T must be positive")
        a = self.a
        if np.isscalar(a):
            a = (float(a), float(a))
        object.__setattr__(self, "a", (float(a[0]), float(a[1])))


@dataclass(frozen=True)
class Stencil:
    """Five-point (2D) / three-point (1D) periodic stencil coefficients.

    (M u)_{i,j} = cc·u_{i,j} + ce·u_{i+1,j} + cw·u_{i−1,j} + cn·u_{i,j+1} + cs·u_{i,j−1}
    (cn = cs = 0 in 1D). The transpose swaps e↔w and n↔s because the central
    first difference is skew and the Laplacian symmetric (`problems.py:319-322`).
    """

    cc: float
    ce: float
    cw: float
    cn: float
    cs: float

    def transpose(self) -> "Stencil":
        return Stencil(self.cc, self.cw, self.ce, self.cs, self.cn)

    def as_tuple(self) -> tuple[float, float, float, float, float]:
        return (self.cc, self.ce, self.cw, self.cn, self.cs)


def advdiff_stencil(grid: Grid, a: tuple[float, float], D: float) -> Stencil:
    """A = −a_x∂x − a_y∂y + D∇², central differences (`problems.py:106-152`)."""
    ax, ay = a
    hx = grid.hx
    ce = -ax / (2.0 * hx) + D / (hx * hx)
    cw = ax / (2.0 * hx) + D / (hx * hx)
    cc = -2.0 * D / (hx * hx)
    cn = cs = 0.0
    if grid.dim == 2:
        hy = grid.hy
        cn = -ay / (2.0 * hy) + D / (hy * hy)
        cs = ay / (2.0 * hy) + D / (hy * hy)
        cc += -2.0 * D / (hy * hy)
    return Stencil(cc, ce, cw, cn, cs)


def diffusion_stencil(grid: Grid, D: float) -> Stencil:
    """D∇² alone: the constant linear part of Burgers (`problems.py:197-210`)."""
    return advdiff_stencil(grid, (0.0, 0.0), D)


# ---------------------------------------------------------------------------
# Fourier control basis (time-constant control f = Σ c_k φ_k)
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class ModeBasis:
    """Separable Fourier basis φ_k(x, y) = X_{ix[k]}(x) · Y_{iy[k]}(y).

    1D, K modes: pairs {cos(m x), sin(m x)}, m = 1..K/2.
    2D, K = 4M² modes: {cos,sin}(m_x x)·{cos,sin}(m_y y), m_x, m_y = 1..M, in
    the order (m_x, m_y, [cc, cs, sc, ss]).
    ``tx`` (rows × nx) and ``ty`` (rows × ny) hold the 1D factor tables; the
    device evaluates φ_k from them, never a K×n matrix.
    """

    K: int
    tx: np.ndarray = field(repr=False)
    ty: np.ndarray = field(repr=False)
    ix: np.ndarray = field(repr=False)
    iy: np.ndarray = field(repr=False)

    def field(self, coeffs: np.ndarray) -> np.ndarray:
        """f = Σ_k c_k φ_k on the flat grid; ``coeffs`` (..., K) → (..., n)."""
        c = np.asarray(coeffs, dtype=np.float64)
        phi = self.matrix()
        return c @ phi

    def project(self, G: np.ndarray) -> np.ndarray:
        """⟨φ_k, G⟩ for (..., n) → (..., K) (plain, unweighted inner product)."""
        return np.asarray(G) @ self.matrix().T

    def matrix(self) -> np.ndarray:
        """Dense K×n basis (host-side helper for small grids and tests)."""
        ny, nx = self.ty.shape[1], self.tx.shape[1]
        out = np.empty((self.K, ny * nx))
        for k in range(self.K):
            out[k] = np.outer(self.ty[self.iy[k]], self.tx[self.ix[k]]).ravel()
        return out


@dataclass(frozen=True)
class FieldBasis:
    """The control as a full spatial field (K = n, the reference's forcing field f_spatial,
    `problems.py:155-162`): ``field`` and ``project`` are the identity, and the gradient is the
    field ∂J/∂f itself. The device runs it with PX_FLAG_FIELD_CONTROL (no factor tables)."""

    K: int
    tx: np.ndarray = field(default_factory=lambda: np.ones((1, 1)), repr=False)
    ty: np.ndarray = field(default_factory=lambda: np.ones((1, 1)), repr=False)
    ix: np.ndarray = field(default_factory=lambda: np.zeros(1, dtype=np.int32), repr=False)
    iy: np.ndarray = field(default_factory=lambda: np.zeros(1, dtype=np.int32), repr=False)

    is_field = True

    def field(self, coeffs: np.ndarray) -> np.ndarray:
        return np.asarray(coeffs, dtype=np.float64)

    def project(self, G: np.ndarray) -> np.ndarray:
        return np.asarray(G, dtype=np.float64)

    def matrix(self) -> np.ndarray:
        return np.eye(self.K)


def mode_basis(grid: Grid, K: int) -> ModeBasis:
    x = grid.x1()
    if grid.dim == 1:
        if K % 2 or K < 2:
            raise ValueError("1D mode count K must be a positive even number")
        M = K // 2
        tx = np.empty((2 * M, grid.nx))
        for m in range(1, M + 1):
            tx[2 * (m - 1)] = np.cos(m * x)
            tx[2 * (m - 1) + 1] = np.sin(m * x)
        ty = np.ones((1, 1))
        ix = np.arange(K, dtype=np.int32)
        iy = np.zeros(K, dtype=np.int32)
        return ModeBasis(K, tx, ty, ix, iy)
    M = int(round(np.sqrt(K / 4)))
    if 4 * M * M != K:
        raise ValueError("2D mode count K must be 4·M² (cos/sin pairs per axis)")
    y = grid.y1()
    tx = np.empty((2 * M, grid.nx))
    ty = np.empty((2 * M, grid.ny))
    for m in range(1, M + 1):
        tx[2 * (m - 1)] = np.cos(m * x)
        tx[2 * (m - 1) + 1] = np.sin(m * x)
        ty[2 * (m - 1)] = np.cos(m * y)
        ty[2 * (m - 1) + 1] = np.sin(m * y)
    ix = np.empty(K, dtype=np.int32)
    iy = np.empty(K, dtype=np.int32)
    k = 0
    for mx in range(M):
        for my in range(M):
            for sx in range(2):
                for sy in range(2):
                    ix[k] = 2 * mx + sx
                    iy[k] = 2 * my + sy
                    k += 1
    return ModeBasis(K, tx, ty, ix, iy)


# ---------------------------------------------------------------------------
# Spectral enclosures for the exponential-action planner
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class SpectralRegion:
    """A compact set containing the spectrum (or field of values) of an operator.

    ``ellipses``: Minkowski sum of axis-aligned ellipses (center, semi_re,
    semi_im) — exact for the circulant advection–diffusion operator, whose
    1D eigenvalues λ(θ) = D(2cosθ−2)/h² − i·a·sinθ/h trace such an ellipse
    and whose 2D eigenvalues are sums of the two axes' (normal operator).
    ``rect``: (re_lo, re_hi, im) box bounding the field of values of a
    non-normal operator (the frozen Burgers adjoint).
    ``crouzeix``: 1 for normal operators; 1+√2 (Crouzeix–Palencia) when the
    region bounds the field of values of a non-normal one.
    """

    ellipses: tuple[tuple[float, float, float], ...] = ()
    rect: tuple[float, float, float] | None = None
    crouzeix: float = 1.0

    def box(self) -> tuple[float, float, float]:
        if self.rect is not None:
            return self.rect
        c = sum(e[0] for e in self.ellipses)
        a = sum(e[1] for e in self.ellipses)
        b = sum(e[2] for e in self.ellipses)
        return (c - a, c + a, b)

    def boundary(self, npts: int = 2048) -> np.ndarray:
        """Points on the region's boundary (max-modulus principle: errors of
        analytic functions peak there)."""
        if self.rect is not None:
            lo, hi, im = self.rect
            k = npts // 4
            t = np.linspace(0.0, 1.0, k, endpoint=False)
            return np.concatenate([
                lo + (hi - lo) * t - 1j * im,
                hi + 1j * (-im + 2 * im * t),
                hi - (hi - lo) * t + 1j * im,
                lo + 1j * (im - 2 * im * t),
            ])
        # outward normal angle ψ; each ellipse's support point for that normal
        psi = np.linspace(0.0, 2 * np.pi, npts, endpoint=False)
        z = np.zeros(npts, dtype=np.complex128)
        for c, a, b in self.ellipses:
            t = np.arctan2(b * np.sin(psi), a * np.cos(psi))
            z += c + a * np.cos(t) + 1j * b * np.sin(t)
        return z


def advdiff_region(grid: Grid, a: tuple[float, float], D: float) -> SpectralRegion:
    """Exact spectral enclosure of the periodic central-difference A (and Aᵀ)."""
    ax, ay = a
    hx = grid.hx
    ell = [(-2.0 * D / hx**2, 2.0 * D / hx**2, abs(ax) / hx)]
    if grid.dim == 2:
        hy = grid.hy
        ell.append((-2.0 * D / hy**2, 2.0 * D / hy**2, abs(ay) / hy))
    return SpectralRegion(ellipses=tuple(ell), crouzeix=1.0)


def round_toward(x: float, up: bool, bits: int = 3) -> float:
    """Round x towards +inf (``up``) or -inf to ``bits`` significant bits.

    Used to stabilise plan-cache keys: bounds computed on CPU and GPU that
    differ only by rounding land on the same quantised value.
    """
    if x == 0.0:
        return 0.0
    mag = abs(x)
    q = 2.0 ** (np.floor(np.log2(mag)) - bits)
    grow = (x > 0) == up
    mag = (np.ceil(mag / q) if grow else np.floor(mag / q)) * q
    return float(np.copysign(mag, x))


def frozen_bounds(ubar: np.ndarray, grid: Grid, D: float) -> tuple[float, float, float]:
    """Raw field-of-values box (re_lo, re_hi, im) of B̄ = J(ū)ᵀ, union over rows of ``ubar``.

    B̄y = Dx(ū∘y) − (Dx ū)∘y + D·L y (`problems.py:316-343` with V = 0). Real
    parts of W(B̄) lie in the Gershgorin interval of the symmetric part
    H = ½(Dx·diag ū − diag ū·Dx) − diag(Dx ū) + D·L, imaginary parts within the
    row-sum bound of the skew part S = ½(Dx·diag ū + diag ū·Dx).
    """
    u = np.asarray(ubar, dtype=np.float64).reshape(-1, grid.nx)
    h = grid.hx
    up = np.roll(u, -1, axis=1)
    um = np.roll(u, 1, axis=1)
    dxu = (up - um) * (1.0 / (2.0 * h))
    dh2 = 2.0 * D / (h * h)
    diag = -dxu - dh2
    rad = (np.abs(up - u) + np.abs(u - um)) * (1.0 / (4.0 * h)) + dh2
    im = (np.abs(up + u) + np.abs(u + um)) * (1.0 / (4.0 * h))
    return float(np.min(diag - rad)), float(np.max(diag + rad)), float(np.max(im))


def frozen_bounds_2d(qbar: np.ndarray, grid: Grid, D: float) -> tuple[float, float, float]:
    """Raw field-of-values box (re_lo, re_hi, im) of B̄ = J(q̄)ᵀ for the two-field Burgers system
    (`problems.py:316-343`), union over the rows of ``qbar`` (…, 2n; U block first).

    B̄(a, b) = (Dx(Ūa) + Dy(V̄a) − (DxŪ)a − (DxV̄)b + D∇²a,  Dx(Ūb) + Dy(V̄b) − (DyŪ)a − (DyV̄)b + D∇²b).
    Real parts of W(B̄) lie in the Gershgorin interval of the symmetric part (advective entries
    (Ū_e − Ū_c)/(4hx) …, the diagonal −DxŪ resp. −DyV̄, the block coupling −½(DxV̄ + DyŪ), D∇²);
    imaginary parts within the row sums of the skew part ((Ū_e + Ū_c)/(4hx) …, ½|DyŪ − DxV̄|)."""
    q = np.asarray(qbar, dtype=np.float64).reshape(-1, 2 * grid.npoints)
    n, nx, ny = grid.npoints, grid.nx, grid.ny
    hx, hy = grid.hx, grid.hy
    U = q[:, :n].reshape(-1, ny, nx)
    V = q[:, n:].reshape(-1, ny, nx)
    Ue, Uw = np.roll(U, -1, axis=2), np.roll(U, 1, axis=2)
    Un, Us = np.roll(U, -1, axis=1), np.roll(U, 1, axis=1)
    Ve, Vw = np.roll(V, -1, axis=2), np.roll(V, 1, axis=2)
    Vn, Vs = np.roll(V, -1, axis=1), np.roll(V, 1, axis=1)
    dUx, dUy = (Ue - Uw) / (2.0 * hx), (Un - Us) / (2.0 * hy)
    dVx, dVy = (Ve - Vw) / (2.0 * hx), (Vn - Vs) / (2.0 * hy)
    dd = 2.0 * D / (hx * hx) + 2.0 * D / (hy * hy)
    rad = ((np.abs(Ue - U) + np.abs(U - Uw)) / (4.0 * hx) + (np.abs(Vn - V) + np.abs(V - Vs)) / (4.0 * hy)
           + dd + 0.5 * np.abs(dVx + dUy))
    im = ((np.abs(Ue + U) + np.abs(U + Uw)) / (4.0 * hx) + (np.abs(Vn + V) + np.abs(V + Vs)) / (4.0 * hy)
          + 0.5 * np.abs(dUy - dVx))
    da, db = -dUx - dd, -dVy - dd
    lo = min(float(np.min(da - rad)), float(np.min(db - rad)))
    hi = max(float(np.max(da + rad)), float(np.max(db + rad)))
    return lo, hi, float(np.max(im))


def frozen_region_from_bounds(re_lo: float, re_hi: float, im: float) -> SpectralRegion:
    """Quantised FOV box → region (Crouzeix–Palencia factor 1+√2).

    Bounds are rounded outward to 3 significant bits so that CPU and GPU slice
    means that differ only by rounding select the same exp-action plan.
    """
    rect = (round_toward(re_lo, up=False), round_toward(re_hi, up=True), round_toward(im, up=True))
    return SpectralRegion(rect=rect, crouzeix=1.0 + np.sqrt(2.0))


def burgers_frozen_region(ubar: np.ndarray, grid: Grid, D: float) -> SpectralRegion:
    """Union FOV region of the frozen adjoint operators J(ū_p)ᵀ over all slices."""
    return frozen_region_from_bounds(*frozen_bounds(ubar, grid, D))
