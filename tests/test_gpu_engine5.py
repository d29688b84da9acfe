"""Engine 5 (pipeline of CTA sets, strips held on chip, pit_newton_ps.cuh) against the oracle.

The all-at-once Newton iteration converges to the solution of the discrete BDF1 system whatever inexact level solver
and whatever schedule it uses (the converged solution equals the sequential one), so the converged
U must match the oracle's sequential solve to 1e-10 (normwise, R17) on every shape class the engine
accepts: constant-viscosity Burgers on periodic grids, 512 or 256 unknowns per row, strips of 20 / 22 (14 / 16) rows
in two row groups per CTA (the upper group with its columns swapped when it starts on an odd row), one to eight CTA
sets, one or several passes of the level pipeline.  Plus: agreement with engine 4 (same sweeps, another schedule),
determinism, the host path, ENOCONV, the reported level-solve residuals.
"""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2406_00878_b200 import pit, workloads as W

from gpu_util import gpu_solve, normwise_rel

pytestmark = pytest.mark.gpu


def _sol(p, **cfg):
    U, hist, nit, st, stats = gpu_solve(p, engine=5, **cfg)
    assert stats["engine"] == 5
    return U, hist, nit, st, stats


def _burgers(nx, ny, nt, dt=1e-4, nu=5e-3, seed=0):
    rng = np.random.default_rng(seed)
    p = W.custom(f"burgers_{nx}x{ny}x{nt}", W.BURGERS, W.PERIODIC, nx, ny, nt, dt, nu, 0.0, u0=np.zeros(nx * ny))
    X, Y = p.grid()
    p.u0 = np.ascontiguousarray((np.sin(2 * np.pi * X + 0.3) * np.sin(4 * np.pi * Y + 0.1) + 0.2 * np.cos(2 * np.pi * Y)
                                 + 1e-3 * rng.standard_normal(X.shape)).reshape(-1))
    return p


# (name, problem, pipeline depth): strips of 22 rows only (44 = 2 x 22), 22 + 22 + 20 (64), 6 strips of 22/20 (128),
# four strips of 22 (88) under 8 sets; 256-wide: 16 + 14 (30), 3 x 16/14 (44); several passes when the depth is
# below the Newton iteration count
CASES = [
    ("burgers_512x44x3_d1", lambda: _burgers(512, 44, 3), 1),
    ("burgers_512x44x5_d2", lambda: _burgers(512, 44, 5), 2),
    ("burgers_512x64x6_d3", lambda: _burgers(512, 64, 6), 3),
    ("burgers_512x128x9_d6", lambda: _burgers(512, 128, 9), 6),
    ("burgers_512x88x4_d8", lambda: _burgers(512, 88, 4), 8),
    ("burgers_256x30x5_d2", lambda: _burgers(256, 30, 5, dt=2e-4), 2),
    ("burgers_256x44x7_d4", lambda: _burgers(256, 44, 7, dt=2e-4), 4),
    ("c5_prefix", lambda: W.config(5, nt=8), 0),
    ("c4_prefix", lambda: W.config(4, nt=12), 0),
    ("c2_full", lambda: W.config(2), 0),                       # 64 unknowns per row: one warp per row group, strips of 4 / 2 rows
]


@pytest.mark.parametrize("name,make,depth", CASES, ids=[c[0] for c in CASES])
def test_engine5_converged_solution_matches_oracle(name, make, depth):
    p = make()
    U, hist, nit, st, stats = _sol(p, pipeline_depth=depth)
    assert st in (pit.PIT_OK, pit.PIT_OK_FLOOR), (st, hist)
    seq = O.solve_sequential(p)
    assert seq.status == 0
    assert normwise_rel(U, seq.U) <= 1e-10, normwise_rel(U, seq.U)
    # hist[0] is the residual of the initial iterate: no solver in it, it must match the oracle's residual
    R0 = O.spacetime_residual(p, np.tile(p.u0, (p.nt, 1)))
    assert abs(hist[0, 1] / np.abs(R0).max() - 1) <= 1e-12
    assert abs(hist[0, 0] / np.sqrt((R0 * R0).mean()) - 1) <= 1e-12


@pytest.mark.parametrize("depth", [1, 2, 6])
def test_engine5_matches_engine4_per_iteration(depth):
    """Same relaxation (omega, sweeps) as engine 4 on another schedule: the per-iteration histories agree to rounding
    (the strips' accumulation order differs), the iteration count and status are the same."""
    p = W.config(5, nt=10)
    U5, h5, n5, s5, st5 = _sol(p, pipeline_depth=depth)
    U4, h4, n4, s4, st4 = gpu_solve(p, engine=4)
    assert st4["engine"] == 4
    assert (n5, s5) == (n4, s4)
    assert normwise_rel(U5, U4) <= 1e-13
    for col in range(4):                   # norms above the rounding floor agree (below it they are rounding noise)
        big = h4[:, col] > 1e-8 * h4[0, col]
        assert np.allclose(h5[big, col], h4[big, col], rtol=1e-5, atol=0), (col, h5[:, col], h4[:, col])
    assert st5["depth"] == depth and st5["steps"] == p.nt * -(-n5 // depth)


def test_engine5_deterministic_and_host_path():
    p = W.config(5, nt=5)
    U1, h1, n1, s1, _ = _sol(p)
    U2, h2, n2, s2, _ = _sol(p)
    assert np.array_equal(U1, U2) and np.array_equal(h1, h2)
    Uh, hh, nh, sh = pit.solve(p, engine=5)
    assert nh == n1 and np.array_equal(Uh, U1)


def test_engine5_is_the_default_where_it_applies():
    p = W.config(5, nt=4)
    U, hist, nit, st, stats = gpu_solve(p)
    assert stats["engine"] == 5 and st in (0, 1)
    q = W.config(2, n=128, nt=4)          # 128 unknowns per row: no engine-5 instantiation, engine 4 takes it
    U, hist, nit, st, stats = gpu_solve(q)
    assert stats["engine"] == 4 and st in (0, 1)
    with pytest.raises(pit.PitError):
        pit.Solver(W.config(1), engine=5)           # 16 unknowns per row: not covered
    U, hist, nit, st, stats = gpu_solve(W.config(3, nt=2))
    assert stats["engine"] == 5 and st in (0, 1)    # the general law on a Dirichlet grid, 256 unknowns per row


def test_engine5_level_residuals_and_history_rows():
    """The measured relative level-solve residuals stay below lin_rtol wherever they are above the rounding floor, and
    iterations run speculatively past the deciding one leave no history rows."""
    p = W.config(5, nt=6)
    s = pit.Solver(p, engine=5, lin_check=1)
    try:
        from gpu_util import dev, torch_cuda
        torch = torch_cuda()
        d_out = torch.empty((p.nt, p.ns), dtype=torch.float64, device="cuda")
        d_hist = torch.full((s.cfg.newton_max, 4), -1.0, dtype=torch.float64, device="cuda")
        d_info = torch.zeros(2, dtype=torch.int32, device="cuda")
        s.solve_device(dev(p.u0), None, None, d_out, d_hist, d_info)
        torch.cuda.synchronize()
        info = s.engine_info()
        nit = int(d_info[0])
        hist = d_hist.cpu().numpy()
    finally:
        s.close()
    assert info["engine"] == 5 and info["sweeps"] >= 1 and 1.0 <= info["omega"] < 2.0
    assert len(info["linres"]) == nit
    for rel, mx in info["linres"]:
        assert rel <= 1e-6 or mx <= 1e-15, info["linres"]
    assert np.all(hist[:nit] > 0) and np.all(hist[nit:] == 0)


def test_engine5_enoconv_and_sweeps_override():
    p = W.config(4, nt=6)
    U, hist, nit, st, _ = _sol(p, newton_max=2)
    assert st == pit.PIT_ENOCONV and nit == 2 and len(hist) == 2
    U, hist, nit, st, _ = _sol(p, lin_sweeps=1)        # one sweep per level: inexact, more Newton iterations
    U2, hist2, nit2, st2, _ = _sol(p)
    assert st in (0, 1) and nit >= nit2 and normwise_rel(U, U2) <= 1e-10


def test_engine5_repeated_solves_on_one_handle():
    """The second solve on a handle writes its probable final iterate straight into u_out (the ring slot the previous
    solve ended in) and reads the broadcast u^0 instead of a materialised U_0: same bits as the first solve; when the
    iteration count changes (other data: the guess of the slot is wrong) the result equals a fresh handle's; a
    caller's guess goes through ring buffer 0 as before."""
    from gpu_util import dev, torch_cuda
    torch = torch_cuda()
    p = W.config(5, nt=6)
    s = pit.Solver(p, engine=5)

    def run(solver, u0, guess=None):
        d_out = torch.full((p.nt, p.ns), float("nan"), dtype=torch.float64, device="cuda")
        d_hist = torch.zeros((solver.cfg.newton_max, 4), dtype=torch.float64, device="cuda")
        d_info = torch.zeros(2, dtype=torch.int32, device="cuda")
        solver.solve_device(dev(u0), None, None if guess is None else dev(guess), d_out, d_hist, d_info)
        torch.cuda.synchronize()
        return d_out.cpu().numpy(), d_hist.cpu().numpy(), d_info.cpu().tolist()

    try:
        U1, h1, i1 = run(s, p.u0)
        U2, h2, i2 = run(s, p.u0)
        assert i1 == i2 and i1[1] in (0, 1)
        assert np.array_equal(U1, U2) and np.array_equal(h1, h2)
        u0b = 0.25 * p.u0                                   # weaker nonlinearity: fewer iterations than the slot guess
        U3, h3, i3 = run(s, u0b)
        U4, h4, i4 = run(s, p.u0, guess=U1)                 # converged guess: one iteration
        s2 = pit.Solver(p, engine=5)
        try:
            U3f, h3f, i3f = run(s2, u0b)
        finally:
            s2.close()
        assert i3 == i3f and np.array_equal(U3, U3f) and np.array_equal(h3, h3f)
        assert i4[1] in (0, 1) and i4[0] <= 2 and normwise_rel(U4, U1) <= 1e-12
    finally:
        s.close()


# ---- the general law (nonlinear heat) on Dirichlet and periodic grids: pit_newton_ps0.cuh ----------------------------
def _heat(nxu, nyu, nt, bc, dt=5e-4, ring_fn=None, seed=1):
    rng = np.random.default_rng(seed)
    if bc == W.DIRICHLET:
        p = W.custom(f"heat_dir_{nxu}x{nyu}x{nt}", W.HEAT, W.DIRICHLET, nxu + 1, nyu + 1, nt, dt, 1.0, 1.0, u0=np.zeros(nxu * nyu))
    else:
        p = W.custom(f"heat_per_{nxu}x{nyu}x{nt}", W.HEAT, W.PERIODIC, nxu, nyu, nt, dt, 1.0, 1.0, u0=np.zeros(nxu * nyu))
    X, Y = p.grid()
    base = np.sin(np.pi * X) * np.sin(2 * np.pi * Y) + 0.3 * np.cos(2 * np.pi * X) * np.sin(np.pi * Y)
    p.u0 = np.ascontiguousarray((base + 1e-3 * rng.standard_normal(X.shape)).reshape(-1))
    if ring_fn is not None:
        p.ring = W.ring_from(p, ring_fn)
    return p


HEAT_CASES = [
    # Dirichlet: 24 rows = 12 + 12 (two strips), 44 = 12 + 12 + 10 + 10, homogeneous and time-dependent rings
    ("heat_dir_256x24x4_d2", lambda: _heat(256, 24, 4, W.DIRICHLET), 2),
    ("heat_dir_256x44x5_d3", lambda: _heat(256, 44, 5, W.DIRICHLET), 3),
    ("heat_dir_ring_256x44x4_d2", lambda: _heat(256, 44, 4, W.DIRICHLET, ring_fn=lambda x, y, t: 0.2 * np.cos(3 * x + 2 * y) * (1 + 5 * t)), 2),
    ("heat_per_256x44x4_d2", lambda: _heat(256, 44, 4, W.PERIODIC), 2),
    ("c3_prefix", lambda: W.config(3, nt=3), 0),
]


@pytest.mark.parametrize("name,make,depth", HEAT_CASES, ids=[c[0] for c in HEAT_CASES])
def test_engine5_general_law_matches_oracle(name, make, depth):
    p = make()
    U, hist, nit, st, stats = _sol(p, pipeline_depth=depth)
    assert st in (pit.PIT_OK, pit.PIT_OK_FLOOR), (st, hist)
    seq = O.solve_sequential(p)
    assert seq.status == 0
    assert normwise_rel(U, seq.U) <= 1e-10, normwise_rel(U, seq.U)
    U4, h4, n4, s4, st4 = gpu_solve(p, engine=4)
    assert st4["engine"] == 4 and n4 == nit and normwise_rel(U, U4) <= 1e-12


def test_engine5_host_path_streams_the_solution_out():
    """pit_solve on a handle that has solved before copies the probable final iterate to the host level by level while
    the kernel runs (the copy stream follows the strips' level counters): same bits as the first solve's copy after the
    kernel; a changed iteration count (other data) falls back to the copy after the solve and is still right."""
    p = W.config(5, nt=24)
    s = pit.Solver(p, engine=5)
    try:
        U1, h1, n1, s1 = s.solve_host(p.u0, None)
        U2, h2, n2, s2 = s.solve_host(p.u0, None)          # streamed
        assert (n1, s1) == (n2, s2) and s1 in (0, 1)
        assert np.array_equal(U1, U2) and np.array_equal(h1, h2)
        U3, h3, n3, s3 = s.solve_host(0.25 * p.u0, None)    # guess of the final iterate may be wrong
        U4, h4, n4, s4 = s.solve_host(0.25 * p.u0, None)
        assert (n3, s3) == (n4, s4) and np.array_equal(U3, U4)
    finally:
        s.close()
    q = W.custom("quarter", p.pde, p.bc, p.nx, p.ny, p.nt, p.dt, p.m0, p.m2, u0=0.25 * p.u0)
    Uq, hq, nq, sq = pit.solve(q, engine=5)
    assert nq == n3 and np.array_equal(Uq, U3)
