"""The five BASELINE.json configs as seeded synthetic problems.

BASELINE leaves several inputs unspecified; they are fixed here once (SURVEY.md
§8(d), Appendix A) and used identically by the CUDA path, the CPU oracle and the
bench:

* seeds: ``20040546 + 100·config + member`` with ``numpy.random.default_rng``
  (the reference's RNG convention, e.g. `test_paraexp.py:88`); "N(0, σ)" means
  standard deviation σ;
* control: f = Σ_k c_k φ_k, time-constant; 1D basis {cos mx, sin mx}, 2D basis
  {cos,sin}(m_x x)·{cos,sin}(m_y y) (``problems.mode_basis``);
* objective: J = ½‖u(T) − u_target‖² for every config (terminal), u_target a
  seeded smooth field (8 modes in 1D, 16 modes in 2D);
* slice rule n_p = ⌈Δ/dt⌉ (``partition.slice_steps``);
* config 2 descent step lr = 1/(T²·n) (the Hessian of J in the low modes is
  ≈ T²·n/2 because ∂u(T)/∂c_k ≈ T·φ_k); config 3 exp-action tol 1e-12;
  config 5's "10 gradient evaluations" are 10 repeated evaluations of one control;
* configs 4 and 5 (the multi-GPU cases) read their exp-action tol 1e-10 as the error budget of
  the whole sweep's carries (``horizon`` = T): each slice carry is planned to tol/(10·P), so
  the 1-GPU scan and every G-GPU block-scan agree to well below 1e-10.

``scaled(cfg, ...)`` shrinks a config for tests while keeping its structure.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, replace

import numpy as np

from .expaction import ChebyshevConfig, KrylovConfig
from .partition import slice_steps
from .problems import ADVECTION_DIFFUSION, BURGERS, Grid, ProblemSpec, mode_basis
from .systems import System, build_system

SEED_BASE = 20040546


def seed(config: int, member: int) -> int:
    return SEED_BASE + 100 * config + member


@dataclass(frozen=True)
class BaselineCase:
    index: int
    name: str
    grid: Grid
    spec: ProblemSpec
    K: int
    P: int
    dt: float
    expaction: ChebyshevConfig | KrylovConfig
    batch: int = 1
    descent_steps: int = 0
    lr: float = 0.0
    evaluations: int = 1
    target_modes: int = 8

    @property
    def system(self) -> System:
        return build_system(self.grid, self.spec, self.K)

    @property
    def nsteps(self) -> int:
        return slice_steps(self.spec.T / self.P, self.dt)

    @property
    def n(self) -> int:
        return self.grid.npoints

    @property
    def gradients_per_run(self) -> int:
        steps = max(self.descent_steps, 1)
        return self.batch * steps if self.descent_steps else self.batch * self.evaluations

    def inputs(self) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
        """(u0 (n,), u_target (n,), ctrl (B, K)) — deterministic."""
        return make_inputs(self)


def _gaussian_2d(grid: Grid, sigma: float, cx: float, cy: float) -> np.ndarray:
    x, y = grid.coordinates()
    return np.exp(-((x - cx) ** 2 + (y - cy) ** 2) / (2.0 * sigma * sigma))


def make_inputs(c: BaselineCase):
    grid = c.grid
    x = grid.x1()
    idx = c.index
    # control coefficients, one member per batch entry
    std = 0.1 if grid.dim == 1 else 0.05
    ctrl = np.stack([np.random.default_rng(seed(idx, b)).normal(0.0, std, c.K) for b in range(c.batch)])
    # target: seeded smooth field
    tb = mode_basis(grid, c.target_modes)
    tcoef = np.random.default_rng(seed(idx, 50)).normal(0.0, std, c.target_modes)
    u_target = tb.field(tcoef)
    if c.spec.kind == BURGERS:
        rng = np.random.default_rng(seed(idx, 60))
        a = rng.normal(0.0, 1.0, 4)
        b = rng.normal(0.0, 1.0, 4)
        pert = sum(a[m - 2] * np.cos(m * x) + b[m - 2] * np.sin(m * x) for m in range(2, 6))
        pert = 0.05 * pert / np.max(np.abs(pert))
        u0 = 0.5 * np.sin(x) + pert
    elif grid.dim == 1:
        u0 = np.exp(-((x - np.pi) ** 2) / 0.1)
    else:
        if idx == 5:
            off = 0.1 * np.random.default_rng(seed(idx, 60)).normal(0.0, 1.0, 2)
        else:
            off = np.zeros(2)
        u0 = _gaussian_2d(grid, 0.2, np.pi + off[0], np.pi + off[1])
    return u0.astype(np.float64), u_target.astype(np.float64), ctrl.astype(np.float64)


def baseline(index: int) -> BaselineCase:
    """BASELINE.json ``configs[index-1]`` (1-based like the survey's C1..C5)."""
    if index == 1:
        return BaselineCase(1, "c1_advdiff1d_n256", Grid(256), ProblemSpec(ADVECTION_DIFFUSION, (1.0, 0.0), 0.01, 1.0),
                            K=8, P=4, dt=1e-3, expaction=ChebyshevConfig(tol=1e-12))
    if index == 2:
        n = 4096
        T = 2.0
        return BaselineCase(2, "c2_advdiff1d_n4096_b16", Grid(n),
                            ProblemSpec(ADVECTION_DIFFUSION, (1.0, 0.0), 0.005, T),
                            K=32, P=64, dt=2.5e-4, expaction=ChebyshevConfig(tol=1e-12), batch=16,
                            descent_steps=20, lr=1.0 / (T * T * n))
    if index == 3:
        return BaselineCase(3, "c3_burgers1d_n2048", Grid(2048), ProblemSpec(BURGERS, (0.0, 0.0), 0.005, 1.0),
                            K=16, P=64, dt=5e-4, expaction=ChebyshevConfig(tol=1e-12))
    if index == 4:
        return BaselineCase(4, "c4_advdiff2d_512_krylov", Grid(512, 512),
                            ProblemSpec(ADVECTION_DIFFUSION, (1.0, 0.5), 1e-3, 1.0),
                            K=64, P=128, dt=2e-4, expaction=KrylovConfig(m=30, tol=1e-10, horizon=1.0),
                            target_modes=16)
    if index == 5:
        return BaselineCase(5, "c5_advdiff2d_2048_p512", Grid(2048, 2048),
                            ProblemSpec(ADVECTION_DIFFUSION, (1.0, 0.5), 5e-4, 1.0),
                            K=256, P=512, dt=5e-5, expaction=ChebyshevConfig(tol=1e-10, horizon=1.0),
                            evaluations=10, target_modes=16)
    raise ValueError("config index must be 1..5")


def scaled(c: BaselineCase, nx: int | None = None, P: int | None = None, steps_per_slice: int | None = None,
           batch: int | None = None, K: int | None = None, T: float | None = None) -> BaselineCase:
    """Shrunk copy for tests: same kind, coefficients per unit length, structure.

    ``steps_per_slice`` fixes dt = (T/P)/steps (default keeps c.dt).
    """
    grid = c.grid
    if nx is not None:
        grid = Grid(nx, nx if c.grid.dim == 2 else 1)
    spec = c.spec if T is None else replace(c.spec, T=T)
    P = P or c.P
    dt = c.dt if steps_per_slice is None else (spec.T / P) / steps_per_slice
    K = K or c.K
    if grid.dim == 2:
        M = int(math.isqrt(K // 4))
        K = 4 * M * M
    ex = c.expaction if c.expaction.horizon <= 0 else replace(c.expaction, horizon=spec.T)
    return replace(c, grid=grid, spec=spec, P=P, dt=dt, K=K, batch=batch or c.batch, expaction=ex,
                   target_modes=min(c.target_modes, K if grid.dim == 1 else 16))
