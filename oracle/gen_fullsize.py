"""Full-size oracle fixtures for BASELINE configs 4 and 5 — TEST INFRASTRUCTURE ONLY.

Runs the CPU oracle (``oracle.config_mode.linear_gradient``, the numpy restatement of the
reference's Paraexp structure with the configs' numerics) once at BASELINE size and commits
what the GPU parity tests compare against (tests/test_gpu_parity.py::test_fullsize_*):

* config 5 (2048², P = 512, Chebyshev, tol 1e-10 as the sweep budget): the single-rank
  summed-chain scan, the GPU's default formulation on one GPU;
* config 4 (512², P = 128, Krylov m = 30): the 4-block block-scan the GPU runs by default
  (``px_set_local_blocks(4)``, one long span per block).

Stored per config (``tests/golden/fullsize_c{4,5}.npz``): J, ∂J/∂c (all K), the L2 norms of
u(T), q†(0) and ∫q† dt, their sums, and every s-th point of each field in both directions
(s = 8 for 2048², 4 for 512²), plus the plan, the formulation, the wall time and the
numpy / scipy versions. The reference itself cannot express these configs,
so the oracle here is the restatement pinned to the reference by tests/test_reference_pin.py.

    python oracle/gen_fullsize.py --config 5      # ≈ 35 min on one core
    python oracle/gen_fullsize.py --config 4      # a few minutes
"""

from __future__ import annotations

import argparse
import os
import platform
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

STRIDE = {4: 4, 5: 8}
WORLD = {4: 4, 5: 1}  # the GPU's default decomposition on one GPU (local blocks)


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


def run(index: int, out: str) -> None:
    import scipy

    from oracle.config_mode import linear_gradient
    from paper_2004_00546_b200 import baseline
    from paper_2004_00546_b200.expaction import plan_for

    c = baseline(index)
    sysm = c.system
    u0, ut, ctrl = c.inputs()
    region = sysm.region()
    delta = c.spec.T / c.P
    sp = plan_for(region, delta, c.expaction)
    lp = lambda span: plan_for(region, span, c.expaction, base_span=delta)
    world = WORLD[index]
    t0 = time.perf_counter()
    r = linear_gradient(c.grid.nx, c.grid.ny, sysm.A.as_tuple(), sysm.basis, c.spec.T, c.P, c.nsteps, u0, ut,
                        ctrl, sp, lp, lp, formulation="scan" if world == 1 else "blockscan", world=world)
    wall = time.perf_counter() - t0
    s = STRIDE[index]
    nx, ny = c.grid.nx, c.grid.ny

    def sub(f):
        return np.ascontiguousarray(np.reshape(f, (ny, nx))[::s, ::s])

    np.savez_compressed(
        out, config=index, J=r.J, grad=r.grad,
        uT_norm=np.linalg.norm(r.uT), qdag0_norm=np.linalg.norm(r.qdag0), G_norm=np.linalg.norm(r.G),
        uT_sum=np.sum(r.uT), qdag0_sum=np.sum(r.qdag0), G_sum=np.sum(r.G),
        uT_sub=sub(r.uT), qdag0_sub=sub(r.qdag0), G_sub=sub(r.G), stride=s,
        formulation="scan" if world == 1 else f"blockscan({world})",
        slice_plan=np.array([sp.substeps, getattr(sp, "degree", getattr(sp, "m", 0))]),
        wall_seconds=wall, numpy=np.__version__, scipy=scipy.__version__, cpu=cpu_model(), threads=1)
    print(f"config {index}: J={r.J[0]:.15e} |grad|={np.linalg.norm(r.grad):.6e} wall {wall:.1f}s -> {out}",
          flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, required=True, choices=[4, 5])
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    for k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ.setdefault(k, "1")
    out = a.out or os.path.join(ROOT, "tests", "golden", f"fullsize_c{a.config}.npz")
    run(a.config, out)


if __name__ == "__main__":
    main()
