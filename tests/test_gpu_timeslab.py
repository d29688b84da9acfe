"""N4 on the GPU: the time-slab pipeline (paper_2406_00878_b200/timeslab.py) with libpit's pit_slab_iterate_device
as the per-slab worker, 2 and 3 slabs on ONE device (ranks as threads of one process: every kernel is an ordinary
launch, the ranks' waits are host-side, carries are device-to-device copies), against the single-handle solve and the
oracle.  PAPER.md:297, 343: the paper's parallelism over time levels; Eq. (7): the recursion
the slabs continue across their boundaries."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2406_00878_b200 import pit, timeslab as TS, workloads as W

from gpu_util import gpu_solve, normwise_rel, torch_cuda

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("kind,world", [("c5_prefix", 2), ("c4_prefix", 3), ("paper_heat", 2)])
def test_gpu_timeslab_matches_single_solve(kind, world):
    torch = torch_cuda()
    p = {"c5_prefix": lambda: W.config(5, nt=8), "c4_prefix": lambda: W.config(4, nt=9),
         "paper_heat": lambda: W.paper_heat(65, nt=10)}[kind]()
    U1, h1, n1, s1, _ = gpu_solve(p, engine=4)
    slabs = TS.split_levels(p.nt, world)

    def rank_fn(g, comm):
        s, e = slabs[g]
        q = TS.slab_problem(p, s, e)
        wk = TS.GpuSlabWorker(q, device=0)
        try:
            U0 = torch.from_numpy(np.tile(p.u0, (q.nt, 1))).cuda()
            r = TS.solve_timeslab(wk, comm, p.nt, p.ns, torch.from_numpy(p.u0).cuda(), U0, newton_tol=p.newton_tol)
            r.U = r.U.cpu().numpy()
            return r
        finally:
            wk.close()
    res = TS.run_threads(world, rank_fn)
    U = np.concatenate([r.U for r in res])
    assert all(r.status in (pit.PIT_OK, pit.PIT_OK_FLOOR) for r in res)
    assert normwise_rel(U, U1) <= 1e-13, normwise_rel(U, U1)
    seq = O.solve_sequential(p)
    assert normwise_rel(U, seq.U) <= 1e-10
    assert abs(res[0].n_iter - n1) <= 1
