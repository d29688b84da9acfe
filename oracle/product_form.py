"""Test-only numpy oracle for the paper's literal decoupled form (Theorem 1 / Eq. (8)) and its
conditioning analysis (§7).  TEST INFRASTRUCTURE ONLY (see oracle/pit_oracle.c header).

Dense, small, obviously correct: matrices are numpy arrays, products are ``@`` and solves are
``numpy.linalg.solve``.  Each function cites the passage it follows.
"""
from __future__ import annotations

import math

import numpy as np


def block_bidiagonal(A_list):
    """The Newton matrix of Eq. (6): diagonal blocks A_i, sub-diagonal -I."""
    L = len(A_list)
    m = A_list[0].shape[0]
    J = np.zeros((L * m, L * m))
    for i, A in enumerate(A_list):
        J[i * m:(i + 1) * m, i * m:(i + 1) * m] = A
        if i > 0:
            J[i * m:(i + 1) * m, (i - 1) * m:i * m] = -np.eye(m)
    return J


def dense_block_solve(A_list, r_list):
    """Brute force: solve Eq. (6) as one dense system (pivoted LAPACK)."""
    J = block_bidiagonal(A_list)
    x = np.linalg.solve(J, np.concatenate(r_list))
    m = A_list[0].shape[0]
    return [x[i * m:(i + 1) * m] for i in range(len(A_list))]


def forward_recursion(A_list, r_list):
    """Eq. (7) applied row by row, i.e. the recursion of Theorem 1's proof
    (PAPER.md:189-204):  du^1 = A_1^{-1} r^1,  du^n = A_n^{-1} (r^n + du^{n-1})."""
    out = []
    prev = np.zeros_like(r_list[0])
    for A, r in zip(A_list, r_list):
        prev = np.linalg.solve(A, r + prev)
        out.append(prev)
    return out


def product_form(A_list, r_list):
    """Left- and right-hand sides of Eq. (8) by the recursions of §5:
    P^1 = A_1, r~^1 = r^1;  P^{n+1} = P^n A_{n+1};  r~^{n+1} = P^n r^{n+1} + r~^n."""
    P = [A_list[0].copy()]
    rt = [r_list[0].copy()]
    for n in range(1, len(A_list)):
        rt.append(P[-1] @ r_list[n] + rt[-1])
        P.append(P[-1] @ A_list[n])
    return P, rt


def product_form_solve(A_list, r_list, diag_scaling=False):
    """Theorem 1: solve every decoupled system P^n dv^n = r~^n independently.
    ``diag_scaling``: the §7 diagonal preconditioner diag(P^n), applied on the left
    (row scaling; R11)."""
    P, rt = product_form(A_list, r_list)
    out = []
    for Pn, rn in zip(P, rt):
        if diag_scaling:
            d = np.diag(Pn).copy()
            out.append(np.linalg.solve(Pn / d[:, None], rn / d))
        else:
            out.append(np.linalg.solve(Pn, rn))
    return out


def count_nonzero_diagonals(M, tol=0.0):
    """Number of distinct diagonals (offsets) of M holding an entry with |m_ij| > tol."""
    ii, jj = np.nonzero(np.abs(M) > tol)
    return len(set((jj - ii).tolist()))


def five_point_pattern(nx, ny, rng=None):
    """A random matrix with the 5-point pattern of the Jacobian blocks:
    offsets {0, +-1, +-nx} on an nx-by-ny interior grid (x fastest), no wrap."""
    rng = np.random.default_rng(0) if rng is None else rng
    n = nx * ny
    A = np.zeros((n, n))
    for j in range(ny):
        for i in range(nx):
            k = j * nx + i
            A[k, k] = 4.0 + rng.uniform(0.5, 1.5)
            if i + 1 < nx: A[k, k + 1] = -rng.uniform(0.5, 1.5)
            if i > 0: A[k, k - 1] = -rng.uniform(0.5, 1.5)
            if j + 1 < ny: A[k, k + nx] = -rng.uniform(0.5, 1.5)
            if j > 0: A[k, k - nx] = -rng.uniform(0.5, 1.5)
    return A


def eq15_lhs(Nt, h, mu):
    """Left side of Eq. (15): ((1 + 8 mu/(N_t h^2)) / (1 + 2 pi^2 mu / N_t))^{N_t},
    the condition-number estimate K of PAPER.md:327-329 with tau = 1/N_t."""
    return ((1.0 + 8.0 * mu / (Nt * h * h)) / (1.0 + 2.0 * math.pi ** 2 * mu / Nt)) ** Nt


def eq15_max_levels(N, mu, c=1.0, eps=1e-16, nt_max=100000):
    """Largest N_t satisfying Eq. (15): eq15_lhs(N_t) < c h^4 / eps with h = 1/N."""
    h = 1.0 / N
    rhs = c * h ** 4 / eps
    best = 0
    for Nt in range(1, nt_max + 1):
        if eq15_lhs(Nt, h, mu) < rhs:
            best = Nt
        else:
            break
    return best


# ---- N3: the paper's own explicit variant ---------------------------------------------

def bandwidths(M, tol=0.0):
    """(lower, upper) bandwidth of M: max i - j and max j - i over entries with |m_ij| > tol."""
    ii, jj = np.nonzero(np.abs(M) > tol)
    if len(ii) == 0:
        return 0, 0
    return int(max(0, (ii - jj).max())), int(max(0, (jj - ii).max()))


def band_lu_nopivot(M, wl, wu):
    """LU factorisation WITHOUT pivoting of a banded matrix with lower/upper bandwidths wl/wu: the paper's
    "standard direct solver for banded matrices without pivoting" (§8).  Doolittle elimination
    in the textbook order: for k = 0..n-1, l_ik = m_ik / m_kk for i = k+1..k+wl, then m_ij -= l_ik m_kj for
    j = k+1..k+wu.  Returns dense (L unit lower, U upper).  No pivoting means a zero pivot yields inf/nan
    (breakdown), exactly like the solver the paper names."""
    A = np.array(M, dtype=np.float64, copy=True)
    n = A.shape[0]
    L = np.eye(n)
    for k in range(n):
        i1 = min(n, k + wl + 1)
        j1 = min(n, k + wu + 1)
        with np.errstate(divide="ignore", invalid="ignore"):
            l = A[k + 1:i1, k] / A[k, k]
        L[k + 1:i1, k] = l
        A[k + 1:i1, k] = 0.0
        A[k + 1:i1, k + 1:j1] -= np.outer(l, A[k, k + 1:j1])
    return L, np.triu(A)


def band_solve_nopivot(L, U, b, wl, wu):
    """Forward substitution with the unit lower band factor, then back substitution with the upper one."""
    n = len(b)
    y = np.array(b, dtype=np.float64, copy=True)
    for k in range(n):
        i1 = min(n, k + wl + 1)
        y[k + 1:i1] -= L[k + 1:i1, k] * y[k]
    x = y
    for k in range(n - 1, -1, -1):
        x[k] /= U[k, k]
        i0 = max(0, k - wu)
        x[i0:k] -= U[i0:k, k] * x[k]
    return x


def explicit_product_solve(A_list, r_list, diag_scaling=True):
    """The paper's explicit form of Theorem 1: P^n and r~^n by the recursions of §5
    (PAPER.md:221-230), the §7 diagonal preconditioner diag(P^n) applied on the left (DESIGN R11),
    and every decoupled system solved by the banded LU without pivoting over P^n's own band."""
    P, rt = product_form(A_list, r_list)
    out = []
    for Pn, rn in zip(P, rt):
        M, b = Pn, rn
        if diag_scaling:
            d = np.diag(Pn).copy()
            M, b = Pn / d[:, None], rn / d
        wl, wu = bandwidths(M)
        L, U = band_lu_nopivot(M, wl, wu)
        out.append(band_solve_nopivot(L, U, b, wl, wu))
    return out
