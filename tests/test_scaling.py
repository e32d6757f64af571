"""Multi-GPU block-scan model (CPU): structure checks with a synthetic profile."""

import pytest

from paper_2004_00546_b200 import baseline, scaled
from paper_2004_00546_b200.scaling import GpuProfile, predict_blockscan, scaling_table


def test_single_gpu_is_the_reference_point():
    c = scaled(baseline(5), nx=64, P=16, steps_per_slice=4, K=16)
    prof = GpuProfile(rk4_direct=1e-5, rk4_adjoint=1.5e-5, term_direct=2e-6, term_adjoint=2.5e-6, fixed=1e-4)
    p1 = predict_blockscan(c, 1, prof)
    assert p1.speedup == pytest.approx(1.0) and p1.breakdown["allreduce"] == 0.0


def test_rk4_dominated_profile_scales_almost_linearly():
    c = scaled(baseline(5), nx=64, P=16, steps_per_slice=4, K=16)
    prof = GpuProfile(rk4_direct=1e-3, rk4_adjoint=1e-3, term_direct=1e-12, term_adjoint=1e-12)
    tab = scaling_table(c, prof, (1, 2, 4, 8))
    assert [t.G for t in tab] == [1, 2, 4, 8]
    assert tab[-1].efficiency > 0.95
    assert all(b.speedup > a.speedup for a, b in zip(tab, tab[1:]))


def test_long_spans_bound_the_scan_part():
    """With a scan-only profile the first (direct) and last (adjoint) ranks carry the
    long spans; the prediction names a critical rank and never beats G."""
    c = scaled(baseline(5), nx=64, P=16, steps_per_slice=4, K=16)
    prof = GpuProfile(rk4_direct=1e-12, rk4_adjoint=1e-12, term_direct=1e-6, term_adjoint=1e-6)
    for G in (2, 4, 8):
        p = predict_blockscan(c, G, prof)
        assert p.speedup <= G + 1e-9
        assert p.breakdown["long_direct"] > 0 or p.breakdown["long_adjoint"] > 0
