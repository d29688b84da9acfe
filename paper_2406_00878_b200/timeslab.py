"""N4 — the multi-GPU time-slab pipeline of the all-at-once Newton iteration.

The paper parallelises over time levels, one level per core (§6, §8); on GPUs a level is
spread over a whole device and the horizon is cut into SLABS of consecutive levels, one per rank.  Eq. (7)'s
recursion du^n = A_n^{-1}(r^n + du^{n-1}) couples a slab to its predecessor through exactly two
vectors per Newton iteration: U_k at the level before the slab (its residual's time difference) and du_k of that
level (the carry).  Rank g therefore runs iteration k of its slab as soon as rank g-1 has sent those two levels
(point-to-point send/recv, N_s doubles each), and the ranks form a pipeline: rank g works on iteration k while
rank g-1 already works on iteration k+1.  The only collective is the per-iteration norm reduction (2 sums of
squares + 2 maxima) that feeds the stop rule; it is waited for `depth` iterations later, so it never stalls the
pipeline (depth >= world size keeps every rank busy; iterations past the converged one are speculative and
discarded, exactly like the single-GPU level wavefront).

This module is argument plumbing around a per-slab worker: the GPU worker calls libpit's
pit_slab_iterate_device (engine 4); tests inject the oracle's one-iteration routine as the worker and run the
orchestration over gloo on CPU.  Nothing here does method arithmetic beyond combining the slab norms (sums of
squares, maxima) and applying the library's stop rule (R8).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable, List, Optional, Tuple

import numpy as np


def split_levels(nt: int, world: int) -> List[Tuple[int, int]]:
    """Balanced slabs [s, e] (1-based, inclusive) of levels 1..nt over `world` ranks (first nt % world get one more)."""
    if world < 1 or world > nt:
        raise ValueError("need 1 <= world <= nt")
    base, extra = divmod(nt, world)
    out, s = [], 1
    for g in range(world):
        L = base + (1 if g < extra else 0)
        out.append((s, s + L - 1))
        s += L
    return out


def stop_decision(k: int, dn: float, prev: float, tol: float, newton_max: int, finite: bool) -> int:
    """The library's stop rule (pit.h / DESIGN.md R8): 0 converged, 1 converged at the rounding floor, -4 newton_max
    reached, -5 non-finite norms, 2 continue."""
    if not finite:
        return -5
    if dn <= tol:
        return 0
    if k >= 1 and dn > 0.5 * prev and dn <= 1e3 * tol:
        return 1
    if k + 1 >= newton_max:
        return -4
    return 2


@dataclass
class SlabResult:
    U: object                      # the converged iterate of this rank's slab (worker array type)
    hist: np.ndarray               # [n_iter][4] global { rms R, max|R|, rms dU, max|dU| }
    n_iter: int
    status: int
    iterations_run: int            # including the speculative ones
    slab: Tuple[int, int] = field(default=(0, 0))


def solve_timeslab(worker, comm, nt: int, ns: int, u0, U0_slab, newton_tol: float = 1e-12, newton_max: int = 30,
                   stop_norm: int = 0, depth: Optional[int] = None) -> SlabResult:
    """Run the time-slab pipeline on this rank.

    worker: object with ``iterate(uprev, carry_in, Uk) -> (Uk1, carry_out, slab_hist4)`` for this rank's slab
            (``carry_in`` None = 0; slab_hist4 = the slab's {rms R, max|R|, rms dU, max|dU|} over its own unknowns),
            ``zeros_level()`` and ``last_level(U)`` returning worker arrays, and ``to_numpy(x)``.
    comm:   object with rank/world, ``send(x, dst)``, ``recv(like, src)`` (blocking, worker arrays) and
            ``allreduce_async(sums4) -> handle`` with ``handle.wait() -> sums4`` (SUM for entries 0, 2; MAX for 1, 3).
    u0:     u^0 (worker array; used by rank 0), U0_slab: the initial iterate of this rank's slab.
    """
    rank, world = comm.rank, comm.world
    slabs = split_levels(nt, world)
    s, e = slabs[rank]
    L = e - s + 1
    N = float(nt) * float(ns)
    depth = max(2, world) if depth is None else max(1, depth)
    iters = {0: U0_slab}           # iterate k of this slab (kept while a decision may still select it)
    pending = {}                   # k -> allreduce handle
    hist = []
    decided_status, decided_k = 2, None
    prev_dn = float("inf")
    k = 0
    ran = 0
    while True:
        # resolve decisions up to k - depth before running iteration k (every rank takes the same branch)
        while pending and min(pending) <= k - depth:
            kk = min(pending)
            g = pending.pop(kk).wait()
            h4 = np.array([np.sqrt(g[0] / N), g[1], np.sqrt(g[2] / N), g[3]])
            hist.append(h4)
            dn = h4[2] if stop_norm else h4[3]
            st = stop_decision(kk, dn, prev_dn, newton_tol, newton_max, bool(np.all(np.isfinite(h4))))
            prev_dn = dn
            if st != 2:
                decided_status, decided_k = st, kk
                break
        if decided_k is not None or k >= newton_max:
            if decided_k is None:          # every iteration run; the last pending decisions settle it
                while pending:
                    kk = min(pending)
                    g = pending.pop(kk).wait()
                    h4 = np.array([np.sqrt(g[0] / N), g[1], np.sqrt(g[2] / N), g[3]])
                    hist.append(h4)
                    dn = h4[2] if stop_norm else h4[3]
                    st = stop_decision(kk, dn, prev_dn, newton_tol, newton_max, bool(np.all(np.isfinite(h4))))
                    prev_dn = dn
                    if st != 2:
                        decided_status, decided_k = st, kk
                        break
            else:
                for kk in sorted(pending):  # speculative iterations' reductions: complete them, discard
                    pending[kk].wait()
                pending.clear()
            break
        # iteration k of this slab: inputs from the predecessor slab (rank 0: u^0 and no carry)
        if rank == 0:
            uprev, carry = u0, None
        else:
            uprev = comm.recv(worker.zeros_level(), rank - 1)
            carry = comm.recv(worker.zeros_level(), rank - 1)
        Uk = iters[k]
        Uk1, carry_out, h4 = worker.iterate(uprev, carry, Uk)
        if rank + 1 < world:
            comm.send(worker.last_level(Uk), rank + 1)
            comm.send(carry_out, rank + 1)
        h4 = np.asarray(h4, dtype=np.float64)
        sums = np.array([h4[0] ** 2 * L * ns, h4[1], h4[2] ** 2 * L * ns, h4[3]])
        pending[k] = comm.allreduce_async(sums)
        iters[k + 1] = Uk1
        for old in [kk for kk in iters if kk < k + 1 - depth]:
            del iters[old]
        ran += 1
        k += 1
    kf = decided_k + 1
    return SlabResult(U=iters[kf], hist=np.array(hist[:kf]), n_iter=kf, status=decided_status, iterations_run=ran,
                      slab=(s, e))


# ---- torch.distributed communicator ------------------------------------------------------------------------------

class TorchComm:
    """Point-to-point and the norm reduction over torch.distributed (NCCL between GPUs, gloo on CPU)."""

    def __init__(self, device=None):
        import torch
        import torch.distributed as dist
        self.torch, self.dist = torch, dist
        self.rank, self.world = dist.get_rank(), dist.get_world_size()
        self.device = device

    def send(self, x, dst):
        self.dist.send(x.contiguous(), dst)

    def recv(self, like, src):
        buf = self.torch.empty_like(like)
        self.dist.recv(buf, src)
        return buf

    def allreduce_async(self, sums4):
        t = self.torch.tensor(sums4, dtype=self.torch.float64, device=self.device)
        s = t[[0, 2]].clone()
        m = t[[1, 3]].clone()
        w1 = self.dist.all_reduce(s, op=self.dist.ReduceOp.SUM, async_op=True)
        w2 = self.dist.all_reduce(m, op=self.dist.ReduceOp.MAX, async_op=True)

        class H:
            def wait(_self):
                w1.wait()
                w2.wait()
                return np.array([float(s[0]), float(m[0]), float(s[1]), float(m[1])])
        return H()


# ---- the GPU worker: libpit's pit_slab_iterate_device -------------------------------------------------------------

class GpuSlabWorker:
    """One Newton iteration of a slab on this rank's GPU through the C ABI (engine 4)."""

    def __init__(self, p_slab, device=0, stream=None):
        import torch
        from . import pit
        self.torch = torch
        self.p = p_slab
        self.dev = torch.device("cuda", device)
        self.s = pit.Solver(p_slab, device=device, engine=4, newton_max=1)
        self.ring = None if p_slab.ring is None else torch.from_numpy(p_slab.ring).to(self.dev)
        self.hist = torch.zeros(4, dtype=torch.float64, device=self.dev)
        self.stream = stream

    def zeros_level(self):
        return self.torch.zeros(self.p.ns, dtype=self.torch.float64, device=self.dev)

    def last_level(self, U):
        return U[-1]

    def iterate(self, uprev, carry_in, Uk):
        Uk1 = self.torch.empty_like(Uk)
        cout = self.zeros_level()
        self.s.slab_iterate_device(uprev, carry_in, self.ring, Uk, Uk1, cout, self.hist, None, stream=self.stream)
        return Uk1, cout, self.hist.cpu().numpy()

    def to_numpy(self, x):
        return x.cpu().numpy()

    def close(self):
        self.s.close()


def slab_problem(p, s: int, e: int):
    """The slab [s, e] of problem p as a problem of its own (levels s..e, Dirichlet rings of those levels)."""
    from dataclasses import replace
    ring = None if p.ring is None else np.ascontiguousarray(p.ring[s - 1:e])
    q = replace(p, nt=e - s + 1, ring=ring, name=f"{p.name}[{s}..{e}]")
    q.u0 = p.u0
    return q


# ---- in-process communicator: every rank a thread of one process (one-GPU emulation of the pipeline) ------------

class ThreadComm:
    """Ranks as threads of one process (queues for send/recv, a shared table for the reductions).  Used to run the
    pipeline's orchestration on ONE GPU: each rank's kernels are ordinary launches, no kernel ever waits on
    another rank's kernel (the waits are host-side), so the ranks may share a device."""

    def __init__(self, world):
        import queue
        import threading
        self.world = world
        self.q = {(a, b): queue.Queue() for a in range(world) for b in range(world)}
        self.lock = threading.Condition()
        self.red = {}

    def for_rank(self, rank):
        outer = self

        class R:
            pass
        r = R()
        r.rank, r.world = rank, self.world
        r.send = lambda x, dst: outer.q[(rank, dst)].put(x.clone() if hasattr(x, "clone") else np.array(x, copy=True))
        r.recv = lambda like, src: outer.q[(src, rank)].get()

        def allreduce_async(sums4, _rank=rank):
            key = len([k for k in outer.red if k[1] == _rank])
            with outer.lock:
                outer.red[(key, _rank)] = np.asarray(sums4, dtype=np.float64)
                outer.lock.notify_all()

            class H:
                def wait(_self):
                    with outer.lock:
                        outer.lock.wait_for(lambda: all((key, g) in outer.red for g in range(outer.world)))
                        v = [outer.red[(key, g)] for g in range(outer.world)]
                    return np.array([sum(a[0] for a in v), max(a[1] for a in v), sum(a[2] for a in v), max(a[3] for a in v)])
            return H()
        r.allreduce_async = allreduce_async
        return r


def run_threads(world, fn):
    """fn(rank, comm) on `world` threads; returns the per-rank results (re-raises the first failure)."""
    import threading
    tc = ThreadComm(world)
    out, err = [None] * world, []

    def body(g):
        try:
            out[g] = fn(g, tc.for_rank(g))
        except BaseException as e:      # noqa: BLE001
            err.append(e)
    th = [threading.Thread(target=body, args=(g,)) for g in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if err:
        raise err[0]
    return out
