"""Multi-rank host logic on CPU: world-size-2 (and 3) gloo process groups drive the
product's orchestration (`engine.distributed_gradient`: which buffers are
allreduced, in which phase, and the partial conventions of the C ABI) with a CPU
oracle stand-in per rank. The result must equal the single-rank summed-chain
scan (up to the block-scan's exp-action truncation) and the oracle block-scan.
"""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from tests.conftest import ROOT


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _case():
    from paper_2004_00546_b200 import baseline, scaled
    from paper_2004_00546_b200.expaction import plan_for
    c = scaled(baseline(5), nx=24, P=6, steps_per_slice=4, K=4)
    region = c.system.region()
    ps = plan_for(region, c.spec.T / c.P, c.expaction)
    pl = lambda span: plan_for(region, span, c.expaction, base_span=c.spec.T / c.P)
    return c, ps, pl


def _worker(rank, world, port, out_dir):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.config_mode import OracleRank
    from paper_2004_00546_b200.engine import distributed_gradient
    c, ps, pl = _case()
    u0, ut, ctrl = c.inputs()
    eng = OracleRank(c.grid.nx, c.grid.ny, c.system.A.as_tuple(), c.system.basis, c.spec.T, c.P, c.nsteps,
                     u0, ut, ctrl, ps, pl, rank, world)
    distributed_gradient(eng)
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), **{k: eng.buf[k].numpy() for k in eng.FIELDS})
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_gradient_gloo(world, tmp_path):
    from oracle.config_mode import linear_gradient
    port = _free_port()
    mp.start_processes(_worker, args=(world, port, str(tmp_path)), nprocs=world, start_method="spawn")
    c, ps, pl = _case()
    u0, ut, ctrl = c.inputs()
    A = c.system.A.as_tuple()
    scan = linear_gradient(c.grid.nx, c.grid.ny, A, c.system.basis, c.spec.T, c.P, c.nsteps, u0, ut, ctrl, ps)
    bs = linear_gradient(c.grid.nx, c.grid.ny, A, c.system.basis, c.spec.T, c.P, c.nsteps, u0, ut, ctrl, ps,
                         pl, pl, formulation="blockscan", world=world)
    rel = lambda a, b: float(np.linalg.norm(np.ravel(a) - np.ravel(b)) / np.linalg.norm(np.ravel(b)))
    for r in range(world):
        f = np.load(os.path.join(tmp_path, f"rank{r}.npz"))
        # every rank holds the full, identical result after the allreduces
        assert rel(f["UT"], bs.uT) < 1e-13 and rel(f["UT"], scan.uT) < 1e-10
        assert rel(f["QDAG0"], bs.qdag0) < 1e-13 and rel(f["QDAG0"], scan.qdag0) < 1e-10
        assert rel(f["G"], bs.G) < 1e-13
        assert rel(f["GRAD"], bs.grad) < 1e-12 and rel(f["GRAD"], scan.grad) < 1e-9
        assert abs(f["J"][0] - scan.J[0]) <= 1e-10 * scan.J[0]


def test_rank_blocks_cover_slices_contiguously():
    from paper_2004_00546_b200 import rank_block
    for P in (1, 4, 7, 512):
        for world in (1, 2, 3, 4, 8):
            if world > P:
                with pytest.raises(ValueError):
                    rank_block(P, 0, world)
                continue
            blocks = [rank_block(P, r, world) for r in range(world)]
            assert blocks[0][0] == 0 and blocks[-1][1] == P
            for (a0, a1), (b0, b1) in zip(blocks, blocks[1:]):
                assert a1 == b0 and a1 > a0
            sizes = [b - a for a, b in blocks]
            assert max(sizes) - min(sizes) <= 1


def test_phase_failure_maps_to_collective_failure():
    """A failing phase on a rank surfaces as CollectiveFailure(worker, subproblem, cause)
    (the reference's fail-fast convention, `workers.py:140-160`, `errors.py:39-49`)."""
    from types import SimpleNamespace

    from paper_2004_00546_b200.engine import distributed_gradient
    from paper_2004_00546_b200.errors import CollectiveFailure

    calls = []

    class Fake:
        spec = SimpleNamespace(rank=3, world=4)

        def direct_partial(self, s): calls.append("direct")
        def direct_reduce_fields(self): return []
        def view(self, f): return f
        def finish_direct(self, s): calls.append("finish_direct")
        def adjoint_partial(self, s): raise RuntimeError("boom")
        @staticmethod
        def adjoint_reduce_fields(w=True): return []
        def finish_adjoint(self, s): calls.append("finish_adjoint")

    with pytest.raises(CollectiveFailure) as ei:
        distributed_gradient(Fake(), reduce=lambda ts, g, s: None, agree=lambda code, g: code)
    assert ei.value.worker == 3 and ei.value.subproblem == "adjoint"
    assert isinstance(ei.value.cause, RuntimeError)
    assert calls == ["direct", "finish_direct"]


def _failing_worker(rank, world, port, out_dir, bad_rank, bad_phase):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.config_mode import OracleRank
    from paper_2004_00546_b200.engine import distributed_gradient
    from paper_2004_00546_b200.errors import CollectiveFailure
    c, ps, pl = _case()
    u0, ut, ctrl = c.inputs()
    eng = OracleRank(c.grid.nx, c.grid.ny, c.system.A.as_tuple(), c.system.basis, c.spec.T, c.P, c.nsteps,
                     u0, ut, ctrl, ps, pl, rank, world)
    if rank == bad_rank:
        def boom(stream=None):
            raise MemoryError("injected failure")
        setattr(eng, bad_phase, boom)
    outcome = "ok"
    try:
        distributed_gradient(eng)
    except CollectiveFailure as e:
        outcome = f"{e.worker}|{e.subproblem}|{type(e.cause).__name__}"
    with open(os.path.join(out_dir, f"rank{rank}.txt"), "w") as f:
        f.write(outcome)
    dist.destroy_process_group()


@pytest.mark.parametrize("bad_phase,label", [("direct_partial", "direct"), ("adjoint_partial", "adjoint")])
def test_rank_failure_aborts_every_rank(bad_phase, label, tmp_path):
    """One rank fails before a collective: every rank raises CollectiveFailure naming that rank
    and phase (none is left blocked in the allreduce; the reference's abort of all workers,
    `workers.py:140-160`)."""
    world, bad = 2, 1
    mp.start_processes(_failing_worker, args=(world, _free_port(), str(tmp_path), bad, bad_phase), nprocs=world,
                       start_method="spawn")
    for r in range(world):
        worker, phase, cause = open(os.path.join(tmp_path, f"rank{r}.txt")).read().split("|")
        assert int(worker) == bad and phase == label
        assert cause == ("MemoryError" if r == bad else "RuntimeError")
