"""N4 — the time-slab pipeline's orchestration (paper_2406_00878_b200/timeslab.py) on CPU.

The per-slab worker here is the ORACLE's one-iteration routine (or_allatonce_iteration, test infrastructure), so these
tests check the pipeline logic alone — slab split, the two boundary vectors per iteration (U_k of the level before
the slab and its carry du_k, Eq. (7)), the lagged norm reduction and the stop rule — against the
oracle's single all-at-once solve (same iterates bit for bit: the split changes no arithmetic).  World size 2 over
gloo (torch.distributed, 127.0.0.1) and world sizes 1..4 as threads.
"""
import os
import sys

import numpy as np
import pytest

from oracle import oracle as O
from paper_2406_00878_b200 import timeslab as TS, workloads as W

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


class OracleWorker:
    def __init__(self, p_slab):
        self.p = p_slab

    def zeros_level(self):
        return np.zeros(self.p.ns)

    def last_level(self, U):
        return U[-1]

    def iterate(self, uprev, carry_in, Uk):
        Uk1, cout, sums = O.allatonce_iteration(self.p, np.asarray(uprev), None if carry_in is None else np.asarray(carry_in), Uk)
        n = self.p.nt * self.p.ns
        return Uk1, cout, np.array([np.sqrt(sums[0] / n), sums[1], np.sqrt(sums[2] / n), sums[3]])

    def to_numpy(self, x):
        return np.asarray(x)


def _problem(kind):
    if kind == "burgers":
        return W.config(2, n=12, nt=7)
    return W.paper_heat(8, nt=9)                  # Dirichlet with time-dependent rings


@pytest.mark.parametrize("kind", ["burgers", "heat_rings"])
@pytest.mark.parametrize("world", [1, 2, 3, 4])
def test_timeslab_threads_equal_single_allatonce(kind, world):
    p = _problem(kind)
    ref = O.solve_allatonce(p, tol=p.newton_tol)
    slabs = TS.split_levels(p.nt, world)

    def rank_fn(g, comm):
        s, e = slabs[g]
        q = TS.slab_problem(p, s, e)
        return TS.solve_timeslab(OracleWorker(q), comm, p.nt, p.ns, p.u0, np.tile(p.u0, (q.nt, 1)),
                                 newton_tol=p.newton_tol)
    res = TS.run_threads(world, rank_fn)
    U = np.concatenate([r.U for r in res])
    assert all(r.n_iter == ref.niter and r.status == ref.status for r in res)
    assert np.array_equal(U, ref.U)
    for r in res:
        assert np.allclose(r.hist, ref.hist, rtol=1e-12, atol=1e-300)
        assert r.iterations_run >= r.n_iter


def test_split_levels():
    assert TS.split_levels(10, 3) == [(1, 4), (5, 7), (8, 10)]
    assert TS.split_levels(4, 4) == [(1, 1), (2, 2), (3, 3), (4, 4)]
    with pytest.raises(ValueError):
        TS.split_levels(3, 4)


def _gloo_rank(rank, world, port, kind, out_dir):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        p = _problem(kind)
        s, e = TS.split_levels(p.nt, world)[rank]
        q = TS.slab_problem(p, s, e)

        class TorchOracleWorker(OracleWorker):      # torch CPU tensors on the wire
            def zeros_level(self):
                return torch.zeros(self.p.ns, dtype=torch.float64)

            def last_level(self, U):
                return torch.from_numpy(np.ascontiguousarray(np.asarray(U)[-1]))

            def iterate(self, uprev, carry_in, Uk):
                Uk1, cout, h = super().iterate(np.asarray(uprev), None if carry_in is None else np.asarray(carry_in), Uk)
                return Uk1, torch.from_numpy(cout), h
        r = TS.solve_timeslab(TorchOracleWorker(q), TS.TorchComm(), p.nt, p.ns, torch.from_numpy(p.u0),
                              np.tile(p.u0, (q.nt, 1)), newton_tol=p.newton_tol)
        np.savez(os.path.join(out_dir, f"r{rank}.npz"), U=r.U, hist=r.hist, n=r.n_iter, st=r.status)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind", ["burgers", "heat_rings"])
def test_timeslab_gloo_world2_equals_single_allatonce(kind, tmp_path):
    import socket

    import torch.multiprocessing as mp
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    mp.spawn(_gloo_rank, args=(2, port, kind, str(tmp_path)), nprocs=2, join=True)
    p = _problem(kind)
    ref = O.solve_allatonce(p, tol=p.newton_tol)
    r = [np.load(os.path.join(tmp_path, f"r{g}.npz")) for g in range(2)]
    assert all(int(x["n"]) == ref.niter and int(x["st"]) == ref.status for x in r)
    assert np.array_equal(np.concatenate([x["U"] for x in r]), ref.U)
    assert np.allclose(r[0]["hist"], ref.hist, rtol=1e-12)
