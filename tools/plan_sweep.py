"""Time one config's gradient across exp-action tolerances and local-block counts (one GPU).

    python tools/plan_sweep.py --config 5 --tols 1e-10 1e-13 1e-14 --blocks 1 2 4

Prints one JSON line per (tol, blocks): ms per gradient (CUDA events on the work stream),
the per-phase device ms and launches, and the slice plan (substeps × degree).
"""

import argparse
import json
import os
import sys
from dataclasses import replace

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--tols", type=float, nargs="+", default=[None])
    ap.add_argument("--blocks", type=int, nargs="+", default=[1])
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--variants", nargs="*", default=[], help="kernel variants name=value (_native.VARIANTS)")
    args = ap.parse_args()
    import torch
    from paper_2004_00546_b200 import baseline
    from paper_2004_00546_b200.engine import EngineSpec, ParaexpEngine
    c0 = baseline(args.config)
    u0, ut, ctrl = c0.inputs()
    dev = [torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in (u0, ut, ctrl)]
    for tol in args.tols:
        c = c0 if tol is None else replace(c0, expaction=replace(c0.expaction, tol=tol))
        for lb in args.blocks:
            var = tuple((kv.split("=")[0], int(kv.split("=")[1])) for kv in args.variants)
            eng = ParaexpEngine(EngineSpec(c.system, c.P, c.dt, c.expaction, c.batch, local_blocks=lb, variants=var))
            eng.set_inputs(*dev)
            s = int(torch.cuda.current_stream().cuda_stream)
            for _ in range(2):
                eng.gradient(s, want_fields=False)
            torch.cuda.synchronize()
            eng.timing()
            eng.set_timing(True)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(args.steps):
                eng.gradient(s, want_fields=False)
            e1.record()
            torch.cuda.synchronize()
            eng.set_timing(False)
            ph = eng.timing()
            plan = eng.plans.get(0)
            print(json.dumps({
                "config": args.config, "tol": c.expaction.tol, "local_blocks": eng.local_blocks,
                "variants": dict(var),
                "ms_per_gradient": e0.elapsed_time(e1) / args.steps,
                "slice_plan": None if plan is None else [plan.substeps, getattr(plan, "degree", None)],
                "phases": {k: {"ms": v["ms"] / args.steps, "launches": v["launches"] / args.steps}
                           for k, v in ph.items()},
                "J": float(eng.get(0)[0])}), flush=True)
            eng.close()
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
