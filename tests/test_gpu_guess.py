"""N1: the paper's coarse-grid initial guess on the GPU against the oracle
(oracle/coarse_guess.py: the C oracle's sequential BDF1 on the coarse grid + numpy splines).

The GPU solves the coarse problem with its own all-at-once engine and interpolates with its own spline
kernels; the oracle solves sequentially and interpolates with dense numpy solves.  The two coarse solutions
agree to the Newton tolerance, so the guesses agree to ~1e-11 relative (tolerance 1e-9 normwise)."""
import numpy as np
import pytest

from oracle import coarse_guess as CG
from oracle import oracle as O
from paper_2406_00878_b200 import pit, workloads as W

from gpu_util import dev, gpu_solve, normwise_rel, torch_cuda

pytestmark = pytest.mark.gpu

CASES = {
    "heat_dirichlet_ring": (lambda: W.paper_heat(64, nt=8), 4),
    "burgers_dirichlet_ring": (lambda: W.paper_burgers(63, nt=12), 3),
    "burgers_periodic_c2": (lambda: W.config(2, n=48, nt=12), 3),
    "c5_shape": (lambda: W.config(5, n=128, nt=16), 4),
    "heat_homogeneous_c3": (lambda: W.config(3, n=63, nt=8), 4),
    "one_coarse_level": (lambda: W.paper_heat(32, nt=4), 4),
}


def gpu_guess(p, cf):
    torch = torch_cuda()
    s = pit.Solver(p, guess_cf=cf)
    try:
        d_U0 = torch.empty((p.nt, p.ns), dtype=torch.float64, device="cuda")
        s.initial_guess_device(dev(p.u0), None if p.ring is None else dev(p.ring), d_U0)
        torch.cuda.synchronize()
        return d_U0.cpu().numpy()
    finally:
        s.close()


@pytest.mark.parametrize("case", list(CASES))
def test_guess_matches_oracle(case):
    mk, cf = CASES[case]
    p = mk()
    got = gpu_guess(p, cf)
    ref = CG.coarse_guess(p, cf)
    assert np.isfinite(got).all()
    assert normwise_rel(got, ref) <= 1e-9, normwise_rel(got, ref)


def test_guess_without_coarsening_is_u0_broadcast():
    p = W.config(2, n=16, nt=4)
    torch = torch_cuda()
    s = pit.Solver(p)
    try:
        d_U0 = torch.empty((p.nt, p.ns), dtype=torch.float64, device="cuda")
        s.initial_guess_device(dev(p.u0), None, d_U0)
        torch.cuda.synchronize()
        assert np.array_equal(d_U0.cpu().numpy(), np.tile(p.u0, (p.nt, 1)))
    finally:
        s.close()


@pytest.mark.parametrize("case", ["heat_dirichlet_ring", "burgers_periodic_c2", "c5_shape"])
def test_solve_from_coarse_guess_matches_oracle(case):
    mk, cf = CASES[case]
    p = mk()
    U, hist, nit, st, stats = gpu_solve(p, guess_cf=cf, lin_rtol=1e-13)
    assert st in (0, 1)
    assert stats["guess_ms"] > 0.0
    seq = O.solve_sequential(p)
    assert normwise_rel(U, seq.U) <= 1e-10
    ref = O.solve_allatonce(p, guess=CG.coarse_guess(p, cf))
    assert nit == ref.niter, (nit, ref.niter)
    for k in range(nit):
        for j in range(4):
            if ref.hist[k, j] > 1e-9:
                assert abs(hist[k, j] / ref.hist[k, j] - 1) <= 1e-4, (k, j, hist[k, j], ref.hist[k, j])
    # the coarse guess saves Newton iterations against the u^0 broadcast
    _, _, nit0, _, _ = gpu_solve(p, lin_rtol=1e-13)
    assert nit <= nit0


@pytest.mark.parametrize("kind,nt,expect", [("heat", 8, 2), ("burgers", 12, 3)])
def test_paper_iteration_counts_on_gpu(kind, nt, expect):
    """Tables 3 / 6 (tests/golden/tables3_6_newton_iterations.txt) with the paper's stop test: L2 update norm
    (stop_norm = 1) below 1/10 of the true discretization error."""
    p = W.paper_heat(64, nt=nt) if kind == "heat" else W.paper_burgers(63, nt=nt)
    cf = 4 if kind == "heat" else 3
    e_true = np.sqrt(np.mean((O.solve_sequential(p).U - W.exact_field(p, p.exact)) ** 2))
    U, hist, nit, st, _ = gpu_solve(p, guess_cf=cf, stop_norm=1, newton_tol=0.1 * e_true)
    assert st == 0 and nit == expect, (nit, hist[:, 2], 0.1 * e_true)
    assert hist[nit - 1, 2] <= 0.1 * e_true < hist[nit - 2, 2]


def test_host_path_with_coarse_guess():
    p = W.config(2, n=48, nt=12)
    s = pit.Solver(p, guess_cf=3)
    try:
        U, hist, nit, st = s.solve_host(p.u0)
    finally:
        s.close()
    assert st in (0, 1)
    assert normwise_rel(U, O.solve_sequential(p).U) <= 1e-10


@pytest.mark.parametrize("case", ["periodic", "dirichlet_ring_then_null", "dirichlet_null_then_ring"])
def test_guess_handle_reused_matches_fresh_handle(case):
    """the coarse-march CUDA graph is captured once per handle; a second solve on the same handle (and a
    change of ring presence between calls) must give the U, n_iter and hist of a fresh handle."""
    torch = torch_cuda()
    p, cf = (W.config(2, n=48, nt=12), 3) if case == "periodic" else (W.paper_heat(64, nt=8), 4)
    rings = {"periodic": [None, None], "dirichlet_ring_then_null": [p.ring, None],
             "dirichlet_null_then_ring": [None, p.ring]}[case]

    def run(s, ring):
        d_out = torch.empty((p.nt, p.ns), dtype=torch.float64, device="cuda")
        d_hist = torch.zeros((s.cfg.newton_max, 4), dtype=torch.float64, device="cuda")
        d_info = torch.zeros(2, dtype=torch.int32, device="cuda")
        s.solve_device(dev(p.u0), None if ring is None else dev(ring), None, d_out, d_hist, d_info)
        torch.cuda.synchronize()
        n = int(d_info[0])
        return d_out.cpu().numpy(), d_hist.cpu().numpy()[:n], n
    s = pit.Solver(p, guess_cf=cf)
    try:
        first = run(s, rings[0])
        second = run(s, rings[1])
    finally:
        s.close()
    for got, ring in ((first, rings[0]), (second, rings[1])):
        f = pit.Solver(p, guess_cf=cf)
        try:
            ref = run(f, ring)
        finally:
            f.close()
        assert got[2] == ref[2]
        assert np.array_equal(got[0], ref[0]) and np.array_equal(got[1], ref[1])


def test_host_path_builds_the_coarse_guess():
    """pit_solve (host buffers) with a guess_cf handle starts from the coarse-grid guess like
    pit_solve_device: same n_iter and hist."""
    p = W.paper_heat(64, nt=8)
    U_d, h_d, n_d, s_d, _ = gpu_solve(p, guess_cf=4)
    U_h, h_h, n_h, s_h = pit.solve(p, guess_cf=4)
    assert n_h == n_d and np.array_equal(h_h, h_d) and np.array_equal(U_h, U_d)
    U0, h0, n0, s0, _ = gpu_solve(p)                   # the u^0 start needs more iterations (paper's point)
    assert n0 > n_d
