"""The bench contract's reference arm on the host (no GPU): `bench.py --impl reference` runs the
CPU oracle port of the path on this machine's cores and prints one JSON line with the contract's
keys (the GPU arm's line is checked by the driver on the B200)."""

import json
import os
import subprocess
import sys

from tests.conftest import ROOT


def test_reference_arm_prints_one_contract_line():
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "1",
                        "--steps", "2", "--warmup", "1"], cwd=ROOT, env=env, capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["impl"] == "reference"
    assert d["metric"] == "Paraexp direct-adjoint gradient evals/s" and d["unit"] == "gradient evals/s"
    assert d["higher_is_better"] is True and d["n_gpus"] == 1 and d["steps"] == 2 and d["warmup"] == 1
    assert d["value"] > 0 and d["e2e"]["value"] == d["value"]
    # a full CPU gradient per step: the rate is what the steps' timed seconds say
    assert d["gradient_fraction_per_step"] == 1.0
    assert abs(d["value"] - 1e3 / d["ms_per_step"]) <= 0.5 * d["value"]
    assert d["cpu_baseline"]["host"]["numpy"] and d["cpu_baseline"]["host"]["cpu"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    cb = d["cpu_baseline"]
    assert cb["kind"] == "port" and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    assert d["config"]["workload"]


def test_cpu_reference_full_gradient_matches_oracle():
    """The CPU reference path (every slice solved, W-process block-scan) equals the oracle's
    block-scan restatement, and its sampled-rate model is self-consistent."""
    import numpy as np
    from oracle.config_mode import linear_gradient
    from oracle.cpu_reference import full_gradient, gradient_units, predict_gradient_seconds, sampled_rate
    from paper_2004_00546_b200 import baseline, scaled
    from paper_2004_00546_b200.expaction import plan_for
    from tests.conftest import rel_l2
    c = scaled(baseline(5), nx=48, P=6, steps_per_slice=4, K=16)
    r = full_gradient(c, 3)
    u0, ut, ctrl = c.inputs()
    reg, d = c.system.region(), c.spec.T / c.P
    lp = lambda s: plan_for(reg, s, c.expaction, base_span=d)
    o = linear_gradient(c.grid.nx, c.grid.ny, c.system.A.as_tuple(), c.system.basis, c.spec.T, c.P, c.nsteps,
                        u0, ut, ctrl, plan_for(reg, d, c.expaction), lp, lp, formulation="blockscan", world=3)
    for k, v in (("J", o.J), ("grad", o.grad), ("uT", o.uT), ("qdag0", o.qdag0), ("G", o.G)):
        assert rel_l2(r[k], v) <= 1e-13, k
    rate, wall, units, frac = sampled_rate(c, 2)
    assert rate > 0 and wall > 0 and 0 < frac
    n = gradient_units(c, 0, 2)
    assert n["rk4_direct_step"] == 3 * c.nsteps and n["slice_actions"] == 2
    assert abs(predict_gradient_seconds(c, 2, units) * rate - c.batch) <= 1e-9 * c.batch
