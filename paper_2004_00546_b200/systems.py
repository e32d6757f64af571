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
        return self.grid.npoints

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
        raise ValueError("the Burgers path is 1D (the reference's 2D system with V ≡ 0)")
    return System(grid, spec, mode_basis(grid, K))


def build_field_system(grid: Grid, spec: ProblemSpec) -> System:
    """The linear testbed with the control as a full spatial field (the reference's
    `ProblemSpec.f_spatial`, `problems.py:59-83,155-162`): ∂J/∂f is returned as a field."""
    if spec.kind != ADVECTION_DIFFUSION:
        raise ValueError("field controls: the advection–diffusion testbed (Burgers: tracking.solve_hybrid_tracking)")
    return System(grid, spec, FieldBasis(grid.npoints))
