"""Engine 4 (neighbour-synchronised red-black SOR level solves, pit_newton_nb.cuh) against the oracle.

The all-at-once Newton iteration converges to the solution of the discrete BDF1 system whatever inexact level
solver it uses (the converged solution equals the sequential one), so the converged U must match
the oracle's sequential solve to 1e-10 (normwise, R17) on every shape class the engine accepts:
64..512 unknowns per row, 1..4 rows per CTA, strips of unequal height, both row parities, periodic and Dirichlet
(with time-dependent rings), heat (general law) and Burgers (constant-viscosity law), one or several passes of the
level wavefront.  Plus: the pipeline depth and the residual-check stride do not change the iterates (bitwise), the
run is deterministic, the measured level-solve residuals meet the a-priori bound, ENOCONV after newton_max.
"""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2406_00878_b200 import pit, workloads as W

from gpu_util import gpu_solve, normwise_rel

pytestmark = pytest.mark.gpu


def _sol(p, **cfg):
    U, hist, nit, st, stats = gpu_solve(p, engine=4, **cfg)
    assert stats["engine"] == 4
    return U, hist, nit, st, stats


def _burgers(nx, ny, nt, dt=1e-4, nu=5e-3, seed=0):
    rng = np.random.default_rng(seed)
    p = W.custom(f"burgers_{nx}x{ny}x{nt}", W.BURGERS, W.PERIODIC, nx, ny, nt, dt, nu, 0.0, u0=np.zeros(nx * ny))
    X, Y = p.grid()
    p.u0 = np.ascontiguousarray((np.sin(2 * np.pi * X + 0.3) * np.sin(4 * np.pi * Y + 0.1) + 0.2 * np.cos(2 * np.pi * Y)
                                 + 1e-3 * rng.standard_normal(X.shape)).reshape(-1))
    return p


CASES = [
    # periodic Burgers: rows of 64..512, strips of 1..4 rows (h = nyu / G with G = min(148, nyu)), both parities
    ("burgers_64x64x12", lambda: _burgers(64, 64, 12)),
    ("burgers_128x40x9", lambda: _burgers(128, 40, 9, dt=5e-4)),
    ("burgers_256x150x7", lambda: _burgers(256, 150, 7, dt=2e-4)),
    ("burgers_256x296x5", lambda: _burgers(256, 296, 5, dt=2e-4)),
    ("burgers_512x512x6", lambda: _burgers(512, 512, 6)),
    ("burgers_512x446x5", lambda: _burgers(512, 446, 5)),
    ("c5_prefix", lambda: W.config(5, nt=8)),
    ("c4_prefix", lambda: W.config(4, nt=12)),
    ("c2_full", lambda: W.config(2)),
    # Dirichlet heat, general law (BASELINE c3 recipe), 256 unknowns per row
    ("c3_prefix", lambda: W.config(3, nt=3)),
    ("heat_256x300x3", lambda: W.custom(
        "heat_256x300", W.HEAT, W.DIRICHLET, 257, 301, 3, 5e-4, 1.0, 1.0,
        u0=np.outer(np.sin(np.pi * np.arange(1, 301) / 301), np.sin(np.pi * np.arange(1, 257) / 257)).reshape(-1))),
    # the paper's Table 1 heat problem on a 64-unknown-wide grid: time-dependent Dirichlet rings
    ("paper_heat_65", lambda: W.paper_heat(65, nt=6)),
]


@pytest.mark.parametrize("name,make", CASES, ids=[c[0] for c in CASES])
def test_engine4_converged_solution_matches_oracle(name, make):
    p = make()
    U, hist, nit, st, stats = _sol(p)
    assert st in (pit.PIT_OK, pit.PIT_OK_FLOOR), (st, hist)
    seq = O.solve_sequential(p)
    assert seq.status == 0
    assert normwise_rel(U, seq.U) <= 1e-10, normwise_rel(U, seq.U)
    # hist[0] is the residual of the initial iterate: no solver in it, it must match the oracle's all-at-once mode
    R0 = O.spacetime_residual(p, np.tile(p.u0, (p.nt, 1)))
    assert abs(hist[0, 1] / np.abs(R0).max() - 1) <= 1e-12
    assert abs(hist[0, 0] / np.sqrt((R0 * R0).mean()) - 1) <= 1e-12


def test_engine4_paper_heat_error_matches_table1_protocol():
    """The Table 1 workload class at N = 65 (rings from the exact solution): the discretization error against the
    exact solution equals the oracle's (same discrete solution), a check that the rings enter correctly."""
    p = W.paper_heat(65, nt=65)
    U, hist, nit, st, stats = _sol(p)
    seq = O.solve_sequential(p)
    ex = W.exact_field(p, p.exact)
    assert abs(np.abs(U - ex).max() - np.abs(seq.U - ex).max()) <= 1e-10 * np.abs(ex).max()


@pytest.mark.parametrize("depth", [1, 2, 3])
def test_engine4_depth_and_check_stride_do_not_change_iterates(depth):
    p = W.config(4, nt=10)
    U0, h0, n0, s0, st0 = _sol(p, pipeline_depth=4)
    U1, h1, n1, s1, st1 = _sol(p, pipeline_depth=depth, lin_check=1)
    assert n0 == n1 and s0 == s1
    assert np.array_equal(U0, U1) and np.array_equal(h0, h1)


def test_engine4_deterministic_and_host_path():
    p = W.config(5, nt=5)
    U1, h1, n1, s1, _ = _sol(p)
    U2, h2, n2, s2, _ = _sol(p)
    assert np.array_equal(U1, U2) and np.array_equal(h1, h2)
    Uh, hh, nh, sh = pit.solve(p, engine=4)
    assert nh == n1 and np.array_equal(Uh, U1)


def test_engine4_level_residuals_and_sweep_rule():
    """S = ceil(ln(lin_rtol) / ln(omega - 1)) with Young's omega from the Jacobi bound q of A_1 at U_0; the measured
    relative level-solve residuals ||b - A du||_2 / ||b||_2 of every Newton iteration stay below lin_rtol (the
    a-priori contraction is a bound) wherever the residual is above the rounding floor."""
    p = W.config(5, nt=6)
    s = pit.Solver(p, engine=4, lin_check=1)
    try:
        from gpu_util import dev, torch_cuda
        torch = torch_cuda()
        d_out = torch.empty((p.nt, p.ns), dtype=torch.float64, device="cuda")
        d_hist = torch.zeros((30, 4), dtype=torch.float64, device="cuda")
        d_info = torch.zeros(2, dtype=torch.int32, device="cuda")
        s.solve_device(dev(p.u0), None, None, d_out, d_hist, d_info)
        torch.cuda.synchronize()
        info = s.engine_info()
    finally:
        s.close()
    q = info["q"]
    co = O.jacobian(p, p.u0)
    qref = float(np.max((np.abs(co[1]) + np.abs(co[2]) + np.abs(co[3]) + np.abs(co[4])) / np.abs(co[0])))
    assert abs(q - qref) <= 1e-12 * qref
    qs = 1 - 0.99 * (1 - qref)
    omega = 2 / (1 + np.sqrt(1 - qs * qs))
    assert abs(info["omega"] - omega) <= 1e-14
    assert info["sweeps"] == int(np.ceil(np.log(1e-6) / np.log(omega - 1)))
    for rel, mx in info["linres"]:
        assert rel <= 1e-6 or mx <= 1e-15, info["linres"]


def test_engine4_enoconv_and_sweeps_override():
    p = W.config(4, nt=6)
    U, hist, nit, st, _ = _sol(p, newton_max=2)
    assert st == pit.PIT_ENOCONV and nit == 2 and len(hist) == 2
    U, hist, nit, st, _ = _sol(p, lin_sweeps=1)        # one sweep per level: inexact, more Newton iterations
    U2, hist2, nit2, st2, _ = _sol(p)
    assert st in (0, 1) and nit >= nit2 and normwise_rel(U, U2) <= 1e-10
