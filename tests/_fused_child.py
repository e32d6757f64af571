"""Child process for tests/test_gpu_parity.py::test_fused_two_step_march_forced.

The RK4 march's two-steps-per-launch kernel (k_rk4_march2) is chosen inside the
library from the environment at first use (PX_MARCH2, PX_M2_VAR), so forcing it on
small grids needs a fresh process. Checks several edge shapes against the oracle.
"""

import sys

import numpy as np

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__file__)))

from tests.test_gpu_parity import _check, _gpu_linear, _oracle_linear  # noqa: E402


def main() -> int:
    from paper_2004_00546_b200 import baseline, release_engines, scaled
    cases = [
        dict(nx=40, P=3, steps_per_slice=3, K=4),     # one fused launch per sweep
        dict(nx=40, P=3, steps_per_slice=4, K=4),     # fused + one single-step remainder
        dict(nx=12, P=2, steps_per_slice=7, K=4),     # rows < pipeline depth: bands wrap the torus
        dict(nx=300, P=4, steps_per_slice=11, K=8),   # strips (VAR 3: 240/368 useful columns), partial last
        dict(nx=640, P=8, steps_per_slice=11, K=16),  # several strips + odd remainder
        dict(nx=1026, P=2, steps_per_slice=6, K=8, T=0.05), # uneven strips of the 3-/4-column kernels
    ]
    for kw in cases:
        c = scaled(baseline(5), **kw)
        _check(_gpu_linear(c), _oracle_linear(c))
        release_engines()
        print("ok", kw, flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
