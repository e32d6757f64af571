"""G-invariance of the block-scan at config 5's full size, measured on one GPU.

World-G sharding is emulated: the G ranks' engines run one after another on the one GPU and
their partials are summed as NCCL's allreduce would (`engine.distributed_gradient`'s phases).
Prints, per G, the relative differences of u(T), q†(0), ∂J/∂c and J against G = 1.

    python tools/g_invariance.py [--worlds 1 2 4 8]
"""

import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def run(world: int, c):
    import torch
    from paper_2004_00546_b200.engine import EngineSpec, ParaexpEngine
    u0, ut, ctrl = c.inputs()
    engs = [ParaexpEngine(EngineSpec(c.system, c.P, c.dt, c.expaction, c.batch, r, world)) for r in range(world)]

    def allreduce(fields):
        for f in fields:
            views = [e.device_view(f) for e in engs]
            total = torch.stack(views).sum(0)
            for v in views:
                v.copy_(total)

    for e in engs:
        e.set_inputs(u0, ut, ctrl)
        e.direct_partial()
    allreduce(engs[0].direct_reduce_fields())
    for e in engs:
        e.finish_direct()
        e.adjoint_partial()
    allreduce(engs[0].adjoint_reduce_fields(True))
    for e in engs:
        e.finish_adjoint()
    r = engs[0].results()
    out = {k: np.array(r[k]) for k in ("uT", "qdag0", "grad", "J")}
    for e in engs:
        e.close()
    torch.cuda.empty_cache()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--worlds", type=int, nargs="+", default=[1, 2, 4, 8])
    ap.add_argument("--tol", type=float, default=None, help="Chebyshev tolerance of every plan (default: the config's)")
    ap.add_argument("--long-tol", type=float, default=None,
                    help="tolerance of the block-scan long-span plans (default: the config's)")
    args = ap.parse_args()
    if args.long_tol is not None:
        from dataclasses import replace
        from paper_2004_00546_b200.engine import ParaexpEngine
        from paper_2004_00546_b200.expaction import plan_for
        orig = ParaexpEngine._plan

        def tight(self, region, span):
            base = self.spec.system.spec.T / self.spec.P
            if span > base * 1.5:
                return plan_for(region, span, replace(self.spec.expaction, tol=args.long_tol), base_span=base)
            return orig(self, region, span)
        ParaexpEngine._plan = tight
    from dataclasses import replace as _replace
    from paper_2004_00546_b200 import baseline
    c = baseline(5)
    if args.tol is not None:
        c = _replace(c, expaction=_replace(c.expaction, tol=args.tol))
    base = run(1, c)
    rel = lambda a, b: float(np.linalg.norm(np.ravel(a) - np.ravel(b)) / np.linalg.norm(np.ravel(b)))
    rows = []
    for w in args.worlds:
        if w == 1:
            continue
        r = run(w, c)
        rows.append({"G": w, **{k: rel(r[k], base[k]) for k in base}})
        print(json.dumps(rows[-1]), flush=True)


if __name__ == "__main__":
    main()
