"""(b2) the paper's literal decoupled form on the GPU: Theorem 1 / Eq. (8) with the recursions of
PAPER.md:221-230, inside the Section 7 conditioning window.

Pinned against the dense numpy product-form oracle (oracle/product_form.py: P^m formed with `@`,
numpy.linalg.solve) built from the CPU oracle's Jacobian blocks and residuals, and against the recurrence."""
import numpy as np
import pytest

from oracle import oracle as O
from oracle import product_form as PF
from paper_2406_00878_b200 import pit, workloads as W

from gpu_util import dev, gpu_solve, normwise_rel, torch_cuda

pytestmark = pytest.mark.gpu


def _window_case(p, s0, L, seed):
    torch = torch_cuda()
    rng = np.random.default_rng(seed)
    U = np.tile(p.u0, (p.nt, 1)) + 0.05 * rng.standard_normal((p.nt, p.ns))
    R = O.spacetime_residual(p, U)
    carry = None if s0 == 1 else 0.01 * rng.standard_normal(p.ns)
    s = pit.Solver(p, lin_rtol=1e-13)
    try:
        dU = torch.zeros((L, p.ns), dtype=torch.float64, device="cuda")
        info = torch.zeros(2, dtype=torch.int32, device="cuda")
        s.product_window_device(s0, L, dev(U), dev(p.u0), None if p.ring is None else dev(p.ring), dev(R),
                                None if carry is None else dev(carry), dU, info)
        torch.cuda.synchronize()
        got = dU.cpu().numpy()
    finally:
        s.close()
    A = [O.to_dense(p, O.jacobian(p, U[s0 - 1 + m], n=s0 + m)) for m in range(L)]
    r = [R[s0 - 1 + m].copy() for m in range(L)]
    if carry is not None:
        r[0] = r[0] + carry
    ref = PF.product_form_solve(A, r)
    rec = PF.forward_recursion(A, r)
    # Section 7 amplification: the level solves stop at a relative residual of lin_rtol = 1e-13 and the
    # decoupled right-hand side r~^m carries the chain product A_1..A_{m-1}, so du^m is only accurate to
    # ~ lin_rtol * prod_{i<m} ||A_i||_inf (the dense oracle solves exactly)
    norms = [np.abs(a).sum(axis=1).max() for a in A]
    tol = [max(1e-10, 10 * 1e-13 * float(np.prod(norms[:m]))) for m in range(L)]
    return got, ref, rec, tol


@pytest.mark.parametrize("case", ["c1_whole_horizon", "c2_window_with_carry", "paper_heat_ring"])
def test_product_window_matches_dense_theorem1(case):
    if case == "c1_whole_horizon":
        p, s0, L = W.config(1), 1, 8
    elif case == "c2_window_with_carry":
        p, s0, L = W.config(2, n=12, nt=9), 3, 5
    else:
        p, s0, L = W.paper_heat(10, nt=6), 2, 4
    got, ref, rec, tol = _window_case(p, s0, L, seed=len(case))
    for m in range(L):
        assert normwise_rel(got[m], ref[m]) <= tol[m], (m, normwise_rel(got[m], ref[m]), tol[m])
        assert normwise_rel(got[m], rec[m]) <= tol[m]
    assert normwise_rel(got[0], ref[0]) <= 1e-10   # the first row is a plain level solve


def test_product_form_on_c1_whole_horizon_matches_oracle():
    """c1's whole horizon is inside the Section 7 gate: PRODUCT_WINDOW runs Theorem 1 over all 8 levels as one window
    (AUTO is the level recurrence, asynchronous on the stream; R19)."""
    p = W.config(1)
    U, hist, nit, st, stats = gpu_solve(p, inverse_mode=pit.PIT_INV_PRODUCT_WINDOW, lin_rtol=1e-13)
    assert stats["product_form"]
    assert st in (0, 1)
    seq = O.solve_sequential(p)
    assert normwise_rel(U, seq.U) <= 1e-10
    Ur, hr, nr, sr, str_ = gpu_solve(p, inverse_mode=pit.PIT_INV_RECURRENCE, lin_rtol=1e-13)
    assert not str_["product_form"]
    assert nr == nit
    assert normwise_rel(U, Ur) <= 1e-13
    for k in range(nit):
        for j in range(4):
            if hr[k, j] > 1e-10:
                assert abs(hist[k, j] / hr[k, j] - 1) <= 1e-8


def test_forced_windows_chained_by_the_carry():
    p = W.config(2, n=16, nt=12)
    Ur, hr, nr, sr, _ = gpu_solve(p, inverse_mode=pit.PIT_INV_RECURRENCE)
    Up, hp, npi, sp, stp = gpu_solve(p, inverse_mode=pit.PIT_INV_PRODUCT_WINDOW, window=5)
    assert stp["product_form"] and sp in (0, 1) and npi == nr
    assert normwise_rel(Up, Ur) <= 1e-12


def test_section7_gate_rejects_a_stiff_window():
    """Heat with tau mu / h^2 ~ 0.5 (||A||_inf ~ 5): a 12-level chain multiplies to > 1e6."""
    p = W.config(3, n=32, nt=12)
    with pytest.raises(pit.PitError) as e:
        gpu_solve(p, inverse_mode=pit.PIT_INV_PRODUCT_WINDOW, window=12)
    assert e.value.code == pit.PIT_ECOND
    # the gate-derived windows (window = 0) stay inside the bound and converge to the oracle
    U, hist, nit, st, stats = gpu_solve(p, inverse_mode=pit.PIT_INV_PRODUCT_WINDOW)
    assert st in (0, 1) and stats["product_form"]
    assert normwise_rel(U, O.solve_sequential(p).U) <= 1e-10
