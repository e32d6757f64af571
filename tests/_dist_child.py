"""Child for tests/test_gpu_parity.py::test_two_rank_gloo_on_one_gpu (run under torchrun).

Both ranks share the one GPU; collectives go through gloo (host-mediated: no kernel
waits on another rank). Rank 0 writes J, grad, u(T), q†(0), G as .npy next to argv[1].
"""

import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main() -> int:
    import torch
    import torch.distributed as dist
    from paper_2004_00546_b200 import RK4Config, baseline, direct_adjoint_loop, scaled
    out = sys.argv[1]
    torch.cuda.set_device(0)
    dist.init_process_group("gloo")
    kind = sys.argv[2]
    c = scaled(baseline(5), nx=96, P=12, steps_per_slice=8, K=16) if kind == "c5" else baseline(int(kind))
    u0, ut, ctrl = c.inputs()
    loop = direct_adjoint_loop(c.system, ctrl, ut, "linear" if c.system.is_linear else "hybrid", N=c.P,
                               rk=RK4Config(c.dt), expaction=c.expaction, u0=u0)
    if dist.get_rank() == 0:
        np.savez(out, J=np.ravel(loop.J), grad=np.ravel(loop.grad), uT=loop.direct.final_state,
                 qdag0=loop.adjoint.initial_state, G=loop.adjoint.integral)
    dist.barrier()
    dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
