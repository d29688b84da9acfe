"""Pins of the N3 oracle (oracle/product_form.py): the banded LU without pivoting the paper names
 and the explicit product form of Theorem 1 with the §7 diagonal preconditioner."""
import numpy as np
import pytest

from oracle import product_form as PF


def _banded(n, wl, wu, rng, dominant=True):
    M = np.zeros((n, n))
    for i in range(n):
        for j in range(max(0, i - wl), min(n, i + wu + 1)):
            M[i, j] = rng.uniform(-1.0, 1.0)
        if dominant:
            M[i, i] = np.abs(M[i]).sum() + 1.0
    return M


@pytest.mark.parametrize("n,wl,wu", [(1, 0, 0), (7, 1, 1), (30, 3, 5), (40, 7, 2), (25, 24, 24)])
def test_band_lu_reproduces_the_matrix_and_keeps_the_band(n, wl, wu):
    rng = np.random.default_rng(n * 100 + wl * 10 + wu)
    M = _banded(n, wl, wu, rng)
    L, U = PF.band_lu_nopivot(M, wl, wu)
    assert np.abs(L @ U - M).max() <= 1e-13 * np.abs(M).max()
    assert np.allclose(np.diag(L), 1.0) and np.all(np.triu(L, 1) == 0)
    # no pivoting => no fill outside the band (the property that makes a band solver a band solver)
    lw, _ = PF.bandwidths(L)
    _, uw = PF.bandwidths(U)
    assert lw <= wl and uw <= wu
    b = rng.standard_normal(n)
    x = PF.band_solve_nopivot(L, U, b, wl, wu)
    assert np.abs(x - np.linalg.solve(M, b)).max() <= 1e-12 * max(1.0, np.abs(x).max())


def test_band_lu_matches_scipy_lu_when_no_pivoting_is_needed():
    scipy_linalg = pytest.importorskip("scipy.linalg")
    rng = np.random.default_rng(5)
    M = _banded(20, 3, 3, rng)
    Pm, Ls, Us = scipy_linalg.lu(M)
    assert np.allclose(Pm, np.eye(20))             # diagonally dominant: partial pivoting never swaps
    L, U = PF.band_lu_nopivot(M, 3, 3)
    assert np.abs(L - Ls).max() <= 1e-13 and np.abs(U - Us).max() <= 1e-12


def test_band_lu_without_pivoting_breaks_down_on_a_zero_pivot():
    M = np.array([[0.0, 1.0], [1.0, 1.0]])          # non-singular, but the first pivot is 0
    L, U = PF.band_lu_nopivot(M, 1, 1)
    x = PF.band_solve_nopivot(L, U, np.array([1.0, 2.0]), 1, 1)
    assert not np.all(np.isfinite(x))
    assert np.allclose(np.linalg.solve(M, [1.0, 2.0]), [1.0, 1.0])


def test_product_band_grows_by_nx_per_factor():
    """P^m = A_1..A_m of 5-point blocks has half-bandwidth m*nx (offsets a + b nx, |a| + |b| <= m; Theorem 2,
    PAPER.md:269-278), the band the explicit solver factors."""
    nx, ny = 6, 7
    rng = np.random.default_rng(1)
    A = [PF.five_point_pattern(nx, ny, rng) for _ in range(4)]
    P, _ = PF.product_form(A, [np.zeros(nx * ny)] * 4)
    for m, Pm in enumerate(P, start=1):
        assert PF.bandwidths(Pm) == (min(m * nx, nx * ny - 1), min(m * nx, nx * ny - 1))


@pytest.mark.parametrize("scaling", [True, False])
def test_explicit_product_solve_equals_the_recursion(scaling):
    """Theorem 1: the decoupled systems have the solution of Eq. (6)."""
    nx, ny, L = 5, 4, 5
    rng = np.random.default_rng(7)
    A = [PF.five_point_pattern(nx, ny, rng) / 6.0 for _ in range(L)]
    r = [rng.standard_normal(nx * ny) for _ in range(L)]
    got = PF.explicit_product_solve(A, r, diag_scaling=scaling)
    ref = PF.dense_block_solve(A, r)
    for g, e in zip(got, ref):
        assert np.abs(g - e).max() <= 1e-12 * max(1.0, np.abs(e).max())
