"""Offline validation of the CPU reference arm's bounded sample — TEST INFRASTRUCTURE ONLY.

``bench.py --impl reference`` (and the GPU arm's ``cpu_baseline``) cannot run a full config-4/5
CPU gradient inside the driver's few-minute budget, so it times a bounded sample (every worker
process times each kind of unit on the full-size field) and counts the units of one gradient
(oracle/cpu_reference.py). This script checks that model once: on this host it runs

1. the bounded sample with W workers → the predicted seconds per gradient, and
2. one complete CPU gradient (every slice solved, W-process block-scan) → the measured seconds,

and writes both to ``profiles/r02_cpu_reference_c{k}.json`` (bench.py attaches the file to its
CPU lines as ``validation``). The complete gradient is also compared with the committed
full-size oracle fixture (tests/golden/fullsize_c{k}.npz) when one exists.

    python oracle/time_fullsize_cpu.py --config 4 [--workers 8]
    python oracle/time_fullsize_cpu.py --config 5          # ≈ 1 h on 8 cores
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, required=True, choices=[4, 5])
    ap.add_argument("--workers", type=int, default=os.cpu_count() or 1)
    a = ap.parse_args()
    import numpy as np

    from oracle.cpu_reference import full_gradient, host_info, sampled_rate
    from paper_2004_00546_b200 import baseline
    c = baseline(a.config)
    rate, wall_s, units, frac = sampled_rate(c, a.workers)
    predicted = c.batch / rate
    t0 = time.perf_counter()
    r = full_gradient(c, a.workers)
    measured = time.perf_counter() - t0
    out = {"config": a.config, "workload": c.name, "workers": min(a.workers, c.P),
           "predicted_seconds_per_gradient": predicted, "measured_seconds_per_gradient": measured,
           "predicted_over_measured": predicted / measured, "sample_seconds": wall_s,
           "unit_seconds": units, "host": host_info(),
           "what": "bounded-sample prediction vs one complete CPU gradient (every slice solved, "
                   f"{min(a.workers, c.P)}-process block-scan), same host, same numpy arithmetic"}
    fx = os.path.join(ROOT, "tests", "golden", f"fullsize_c{a.config}.npz")
    if os.path.exists(fx):
        ref = np.load(fx)
        out["vs_fixture"] = {"J_rel": float(np.max(np.abs(r["J"] - ref["J"]) / np.abs(ref["J"]))),
                             "grad_rel_l2": float(np.linalg.norm(r["grad"] - ref["grad"]) / np.linalg.norm(ref["grad"])),
                             "fixture_formulation": str(ref["formulation"])}
    path = os.path.join(ROOT, "profiles", f"r02_cpu_reference_c{a.config}.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
