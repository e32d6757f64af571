"""Host logic of the checkpointed loop (no GPU): schedule, validation, oracle driver."""

import numpy as np
import pytest

from paper_2004_00546_b200 import CheckpointSchedule, MemoryCounter, RK4Config, baseline, run_checkpointed_loop
from paper_2004_00546_b200.errors import ConfigError


def test_schedule_bounds_and_validation():
    s = CheckpointSchedule(1.0, 3)
    assert s.segment_count == 4
    np.testing.assert_allclose(s.times, [0.25, 0.5, 0.75])
    assert s.segment_bounds == [(0.0, 0.25), (0.25, 0.5), (0.5, 0.75), (0.75, 1.0)]
    assert CheckpointSchedule(2.0, 0).segment_bounds == [(0.0, 2.0)]
    with pytest.raises(ValueError):
        CheckpointSchedule(0.0, 1)
    with pytest.raises(ValueError):
        CheckpointSchedule(1.0, -1)


def test_memory_counter_peak():
    m = MemoryCounter()
    m.acquire(5)
    m.release(5)
    m.acquire(3)
    m.acquire(4)
    assert (m.current, m.peak, m.total_allocated) == (7, 7, 12)


def test_run_checkpointed_loop_rejects_bad_inputs():
    c = baseline(3)
    u0, ut, ctrl = c.inputs()
    rk = RK4Config(c.dt)
    with pytest.raises(ConfigError):  # batch > 1
        run_checkpointed_loop(c.system, np.vstack([ctrl, ctrl]), ut, CheckpointSchedule(c.spec.T, 1), "hybrid",
                              N=32, rk=rk)
    with pytest.raises(ValueError):   # algorithm / testbed mismatch
        run_checkpointed_loop(c.system, ctrl, ut, CheckpointSchedule(c.spec.T, 1), "linear", N=32, rk=rk)
    with pytest.raises(ValueError):   # horizon mismatch
        run_checkpointed_loop(c.system, ctrl, ut, CheckpointSchedule(2 * c.spec.T, 1), "hybrid", N=32, rk=rk)
    with pytest.raises(ConfigError):  # no RK4 config
        run_checkpointed_loop(c.system, ctrl, ut, CheckpointSchedule(c.spec.T, 1), "hybrid", N=32)


def test_oracle_checkpoint_driver_m0_is_plain():
    """The oracle's segment walk with M = 0 is exactly one plain gradient."""
    from oracle.config_mode import checkpointed_gradient, linear_gradient
    from paper_2004_00546_b200 import scaled
    from paper_2004_00546_b200.expaction import plan_for
    c = scaled(baseline(1), nx=64, P=4, steps_per_slice=50)
    u0, ut, ctrl = c.inputs()
    plan = plan_for(c.system.region(), c.spec.T / c.P, c.expaction)
    seg = lambda u, qd: linear_gradient(c.grid.nx, c.grid.ny, c.system.A.as_tuple(), c.system.basis, c.spec.T,
                                        c.P, c.nsteps, u, ut, ctrl, plan, qdag_T=qd)
    J, grad, qdag0, G, uT, states = checkpointed_gradient(seg, lambda u: seg(u, None).uT[0], u0, 0)
    ref = seg(u0, None)
    assert np.array_equal(grad, ref.grad) and np.array_equal(qdag0, ref.qdag0) and np.array_equal(G, ref.G)
    assert len(states) == 1
