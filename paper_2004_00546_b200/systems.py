"""Problem bundles: grid + spec + control basis (`pkg/src/paradjoint/systems.py:27-117`).

The reference's `System` carries CSR operators and Python callbacks
(`full_rhs`, `adjoint_apply`, `frozen_adjoint_op`); the CUDA path needs the
*structure* instead — stencil coefficients, the control basis and spectral
enclosures — so that whole sweeps run as kernels.
"""

from __future__ import annotations

from dataclasses import dataclass

from .problems import (
    ADVECTION_DIFFUSION,
    FieldBasis,
    BURGERS,
    Grid,
    ModeBasis,
    ProblemSpec,
    SpectralRegion,
    Stencil,
    advdiff_region,
    advdiff_stencil,
    diffusion_stencil,
    mode_basis,
)


@dataclass(frozen=True)
class System:
    grid: Grid
    spec: ProblemSpec
    basis: ModeBasis

    @property
    def n(self) -> int:
        """State length: the grid's points, twice that for the two-field 2D Burgers system
        (U block first, `problems.py:170-174`)."""
        return self.grid.npoints * (2 if self.is_burgers2d else 1)

    @property
    def is_burgers2d(self) -> bool:
        return self.spec.kind == BURGERS and self.grid.dim == 2

    @property
    def is_linear(self) -> bool:
        return self.spec.kind == ADVECTION_DIFFUSION

    @property
    def A(self) -> Stencil:
        """Constant linear part: full A (advdiff) or D∇² (Burgers), `systems.py:106-117`."""
        if self.is_linear:
            return advdiff_stencil(self.grid, self.spec.a, self.spec.D)
        return diffusion_stencil(self.grid, self.spec.D)

    def region(self) -> SpectralRegion:
        """Spectral enclosure of A (= that of Aᵀ) for the linear testbed."""
        if not self.is_linear:
            raise ValueError("Burgers frozen operators need the direct trajectory")
        return advdiff_region(self.grid, self.spec.a, self.spec.D)


def build_system(grid: Grid, spec: ProblemSpec, K: int) -> System:
    """(`systems.py:106-117`) with a K-mode Fourier control instead of f·sin(ωt)."""
    if spec.kind == BURGERS and grid.dim != 1:
        raise ValueError("mode-basis Burgers is 1D (the reference's 2D system with V ≡ 0); the two-field 2D "
                         "testbed takes field controls: build_burgers2d_system")
    return System(grid, spec, mode_basis(grid, K))


def build_burgers2d_system(grid: Grid, spec: ProblemSpec) -> System:
    """The reference's own Burgers testbed: two fields (U, V) on a 2D grid with a forcing field on
    both components (`problems.py:177-186`, `systems.py:106-117`). It runs the hybrid / serial loop
    with the tracking objective (`tracking.solve_hybrid_tracking`); the control and the gradient
    are fields of length 2·nx·ny."""
    if spec.kind != BURGERS or grid.dim != 2:
        raise ValueError("build_burgers2d_system: a Burgers spec on a 2D grid")
    return System(grid, spec, FieldBasis(2 * grid.npoints))


def build_field_system(grid: Grid, spec: ProblemSpec) -> System:
    """The linear testbed with the control as a full spatial field (the reference's
    `ProblemSpec.f_spatial`, `problems.py:59-83,155-162`): ∂J/∂f is returned as a field."""
    if spec.kind != ADVECTION_DIFFUSION:
        raise ValueError("field controls: the advection–diffusion testbed (Burgers: tracking.solve_hybrid_tracking)")
    return System(grid, spec, FieldBasis(grid.npoints))
