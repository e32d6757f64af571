"""B200-native Paraexp direct-adjoint gradient path (arXiv 2004.00546).

Drop-in for the reference's hot path (`pkg/src/paradjoint`): the
host API keeps the reference's names — problem setup, time partition, the
direct-adjoint loop and the descent driver — and ``backend="cuda"`` runs the
sweeps as hand-written sm_100a fp64 kernels behind the C ABI in
``include/paraexp.h`` (``libparaexp.so``). There is no CPU fallback.
"""

from .checkpointing import (CheckpointRun, CheckpointSchedule, CheckpointTrackingRun, MemoryCounter,
                            run_checkpointed_loop, run_checkpointed_tracking)
from .configs import BaselineCase, baseline, scaled
from .engine import EngineSpec, ParaexpEngine
from .errors import (
    CollectiveFailure,
    ConfigError,
    IntegrationFailure,
    IterationDivergence,
    NativeUnavailable,
    PilotTooShort,
    PropagationFailure,
)
from .expaction import ChebPlan, ChebyshevConfig, KrylovConfig, KrylovPlan, plan_chebyshev, plan_family, plan_krylov
from .hybrid import HybridPlan, TimeLaw, estimate_k, make_hybrid_plan, partition_geometric, slice_offsets
from .nonlinear import NonlinearResult, solve_direct_nonlinear
from .optimization import (
    ALGORITHMS,
    HYBRID,
    LINEAR,
    NONLINEAR,
    AdjointSolution,
    DescentResult,
    DirectSolution,
    LoopResult,
    cost,
    descend,
    direct_adjoint_loop,
    initial_condition_gradient,
    release_engines,
)
from .partition import (
    RK4Config,
    TimePartition,
    WorkerPlan,
    partition_equidistant,
    rank_block,
    slice_steps,
    worker_plans,
)
from .problems import (
    ADVECTION_DIFFUSION,
    BURGERS,
    Grid,
    FieldBasis,
    ModeBasis,
    ProblemSpec,
    SpectralRegion,
    Stencil,
    advdiff_region,
    advdiff_stencil,
    burgers_frozen_region,
    mode_basis,
)
from .solvers import solve_adjoint_linear, solve_direct_linear, solve_hybrid, synthesize_truth
from .systems import System, build_burgers2d_system, build_field_system, build_system
from .tracking import (
    HybridTrackingEngine,
    HybridTrackingResult,
    release_tracking_engines,
    solve_hybrid_tracking,
    solve_nonlinear_tracking,
    synthesize_trajectory,
)

__all__ = [name for name in dir() if not name.startswith("_")]
