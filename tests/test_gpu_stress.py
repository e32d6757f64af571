"""A short, seeded slice of each randomised GPU-vs-oracle sweep (tests/stress_*.py; the long runs are
recorded in DESIGN.md §6) as part of the GPU suite: random shapes, partitions, laws and kernel variants."""

import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("module, count, seed", [
    ("tests.stress_linear", 8, 314),
    ("tests.stress_1d", 8, 315),
    ("tests.stress_tracking", 6, 316),
    ("tests.stress_hybrid1d", 5, 317),
    ("tests.stress_hybrid2d", 6, 318),
])
def test_seeded_random_cases_match_the_oracle(cuda_ok, module, count, seed):
    import importlib
    worst = importlib.import_module(module).run(count, seed)   # a failing case raises after printing it
    assert worst and all(v <= 1e-8 for v in worst.values())
