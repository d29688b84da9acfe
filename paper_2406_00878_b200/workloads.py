"""Seeded synthetic workloads — the ONE module both the oracle side (tests) and the CUDA side use.

It holds problem definitions and initial/boundary DATA only: no residual, Jacobian, solver or any
other arithmetic of the method (that lives, independently, in ``oracle/`` and in ``csrc/``).

Workload recipes:

* ``config(1..5)``: the five BASELINE.json configs.  Seeds ``numpy.random.default_rng(240600878 + c)``,
  draws in the order listed in SURVEY.md §8(d).  Grid convention: ``nx, ny`` are grid INTERVALS
  (R2); BASELINE's "N x N grid" is N x N unknowns, so the Dirichlet configs use
  N + 1 intervals and the periodic configs N intervals.
* ``config(c, nx=.., nt=..)``: the same recipe on a smaller grid / fewer levels (parity-test sizes).
* ``paper_heat(N)`` / ``paper_burgers(N)``: the paper's own accuracy workloads of Tables 1 and 4
   with Dirichlet data from the exact solutions.
* ``heat_exact`` / ``burgers_exact``: the closed-form exact solutions the paper states
  (PAPER.md:374-378 and Eq. (14)); data generators, used for u0 / rings / errors.

There is no public dataset in the paper: every workload is synthetic by construction.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field, replace
from typing import Callable, Optional

import numpy as np

HEAT, BURGERS = 0, 1
DIRICHLET, PERIODIC = 0, 1
SEED_BASE = 240600878


@dataclass
class Problem:
    """One BDF1 space-time problem: the paper's problem statement (Eqs. (1)-(3))."""

    name: str
    pde: int
    bc: int
    nx: int
    ny: int
    nt: int
    x0: float
    x1: float
    y0: float
    y1: float
    dt: float
    m0: float
    m2: float
    newton_tol: float = 1e-12
    u0: np.ndarray = field(default=None, repr=False)      # (ns,) fp64, x fastest
    ring: Optional[np.ndarray] = field(default=None, repr=False)  # (nt, 2(nx+ny)) or None

    @property
    def nxu(self) -> int:
        return self.nx - 1 if self.bc == DIRICHLET else self.nx

    @property
    def nyu(self) -> int:
        return self.ny - 1 if self.bc == DIRICHLET else self.ny

    @property
    def ns(self) -> int:
        return self.nxu * self.nyu

    @property
    def ring_len(self) -> int:
        return 2 * (self.nx + self.ny)

    @property
    def dof(self) -> int:
        return self.ns * self.nt

    @property
    def hx(self) -> float:
        return (self.x1 - self.x0) / self.nx

    @property
    def hy(self) -> float:
        return (self.y1 - self.y0) / self.ny

    def xs(self) -> np.ndarray:
        """x coordinates of the unknown columns."""
        i0 = 1 if self.bc == DIRICHLET else 0
        return self.x0 + (np.arange(self.nxu) + i0) * self.hx

    def ys(self) -> np.ndarray:
        j0 = 1 if self.bc == DIRICHLET else 0
        return self.y0 + (np.arange(self.nyu) + j0) * self.hy

    def grid(self):
        """(X, Y) of the unknown nodes, shape (nyu, nxu)."""
        return np.meshgrid(self.xs(), self.ys(), indexing="xy")

    def with_levels(self, nt: int) -> "Problem":
        ring = None if self.ring is None else self.ring[:nt].copy()
        return replace(self, nt=nt, ring=ring)


def ring_from(prob: Problem, fn: Callable[[np.ndarray, np.ndarray, float], np.ndarray]) -> np.ndarray:
    """Dirichlet ring b(x, y, t^n), n = 1..nt (Eq. (2)), in the ABI's order:
    bottom j=0 (i=0..nx), top j=ny (i=0..nx), left i=0 (j=1..ny-1), right i=nx (j=1..ny-1)."""
    xa = prob.x0 + np.arange(prob.nx + 1) * prob.hx
    yi = prob.y0 + np.arange(1, prob.ny) * prob.hy
    out = np.empty((prob.nt, prob.ring_len))
    for n in range(1, prob.nt + 1):
        t = n * prob.dt
        out[n - 1] = np.concatenate([
            fn(xa, np.full_like(xa, prob.y0), t),
            fn(xa, np.full_like(xa, prob.y1), t),
            fn(np.full_like(yi, prob.x0), yi, t),
            fn(np.full_like(yi, prob.x1), yi, t),
        ])
    return out


# ---- closed-form exact solutions stated by the paper (data generators) -------------------------

def heat_exact(x, y, t, mu0=1e-6, alpha=1.0):
    """u = sqrt( sqrt(alpha/mu0)(x + y) + alpha t + 1 )  (u_ex(x, y, t), R14)."""
    return np.sqrt(np.sqrt(alpha / mu0) * (x + y) + alpha * t + 1.0)


def burgers_exact(x, y, t, mu=1e-3, v=0.5):
    """u = (v/2) [1 - tanh( v (x + y - v t) / (4 mu) )]  (Eq. (14))."""
    return 0.5 * v * (1.0 - np.tanh(v * (x + y - v * t) / (4.0 * mu)))


# ---- BASELINE.json configs -------------------------------------------------------------------

def _u0_c1(p, rng):
    X, Y = p.grid()
    return np.sin(np.pi * X) * np.sin(np.pi * Y)


def _u0_c2(p, rng):
    X, Y = p.grid()
    xi = rng.standard_normal((p.nyu, p.nxu))
    return np.sin(2 * np.pi * X) * np.sin(2 * np.pi * Y) + 1e-3 * xi


def _u0_c3(p, rng):
    X, Y = p.grid()
    u = np.zeros_like(X)
    for _ in range(4):
        a = rng.uniform(0.5, 1.0)
        w = rng.uniform(0.05, 0.15)
        cx = rng.uniform(0.2, 0.8)
        cy = rng.uniform(0.2, 0.8)
        u += a * np.exp(-((X - cx) ** 2 + (Y - cy) ** 2) / (2 * w * w))
    return u


def _u0_c4(p, rng):
    X, Y = p.grid()
    h = p.hx
    xi = rng.standard_normal((p.nyu, p.nxu))
    step = 0.5 * (1 + np.tanh(X / h) - np.tanh((X - 0.5) / h) + np.tanh((X - 1.0) / h))
    return step + 1e-3 * xi


def _u0_c5(p, rng):
    X, Y = p.grid()
    u = np.zeros_like(X)
    for pp in range(1, 9):
        for q in range(1, 9):
            c = rng.standard_normal()
            phi = rng.uniform(0, 2 * np.pi)
            psi = rng.uniform(0, 2 * np.pi)
            u += c * np.sin(2 * np.pi * pp * X + phi) * np.sin(2 * np.pi * q * Y + psi) / (pp * pp + q * q)
    return u


_CONFIGS = {
    # c: (name, pde, bc, N unknowns per direction, nt, dt, m0, m2, u0 recipe)
    1: ("c1_heat_dirichlet_16x16x8", HEAT, DIRICHLET, 16, 8, 1e-3, 1.0, 1.0, _u0_c1),
    2: ("c2_burgers_periodic_64x64x64", BURGERS, PERIODIC, 64, 64, 2e-3, 1e-2, 0.0, _u0_c2),
    3: ("c3_heat_dirichlet_256x256x256", HEAT, DIRICHLET, 256, 256, 5e-4, 1.0, 1.0, _u0_c3),
    4: ("c4_burgers_periodic_256x256x512", BURGERS, PERIODIC, 256, 512, 1e-4, 1e-3, 0.0, _u0_c4),
    5: ("c5_burgers_periodic_512x512x1024", BURGERS, PERIODIC, 512, 1024, 1e-4, 5e-3, 0.0, _u0_c5),
}


def config(c: int, n: Optional[int] = None, nt: Optional[int] = None) -> Problem:
    """BASELINE.json config ``c`` (1..5).  ``n`` overrides the unknowns per direction and ``nt`` the
    number of levels (same recipe and seed; used for parity sizes the oracle finishes quickly)."""
    name, pde, bc, N, NT, dt, m0, m2, recipe = _CONFIGS[c]
    N = N if n is None else n
    NT = NT if nt is None else nt
    intervals = N + 1 if bc == DIRICHLET else N
    if n is not None or nt is not None:
        name = f"{name}@{N}x{N}x{NT}"
    p = Problem(name=name, pde=pde, bc=bc, nx=intervals, ny=intervals, nt=NT,
                x0=0.0, x1=1.0, y0=0.0, y1=1.0, dt=dt, m0=m0, m2=m2, newton_tol=1e-12)
    rng = np.random.default_rng(SEED_BASE + c)
    p.u0 = np.ascontiguousarray(recipe(p, rng).reshape(-1), dtype=np.float64)
    p.ring = None   # homogeneous Dirichlet (c1, c3) / periodic (c2, c4, c5)
    return p


# ---- the paper's own accuracy workloads (Tables 1 and 4) ----------------------------------------

def paper_heat(N: int, mu0: float = 1e-6, alpha: float = 1.0, T: float = 1.0, nt: Optional[int] = None,
               domain=(0.1, 1.1, 0.1, 1.1)) -> Problem:
    """Table 1 protocol: mu = mu0 u^2 on [0.1,1.1]^2, t in [0,1],
    N_t = N_x = N_y = N, u0 and Dirichlet data from the exact solution."""
    nt = N if nt is None else nt
    x0, x1, y0, y1 = domain
    p = Problem(name=f"paper_heat_{N}", pde=HEAT, bc=DIRICHLET, nx=N, ny=N, nt=nt,
                x0=x0, x1=x1, y0=y0, y1=y1, dt=T / nt, m0=0.0, m2=mu0)
    fn = lambda x, y, t: heat_exact(x, y, t, mu0, alpha)
    X, Y = p.grid()
    p.u0 = np.ascontiguousarray(fn(X, Y, 0.0).reshape(-1))
    p.ring = ring_from(p, fn)
    p.exact = fn
    return p


def paper_burgers(N: int, mu: float = 1e-3, v: float = 0.5, T: float = 1.0, nt: Optional[int] = None,
                  domain=(-0.25, 0.75, -0.25, 0.75)) -> Problem:
    """Table 4 protocol: Burgers, mu = 1e-3, v = 0.5, t in [0,1],
    N_t = N_x = N_y = N, on [-0.25,0.75]^2 (R3), data from Eq. (14)."""
    nt = N if nt is None else nt
    x0, x1, y0, y1 = domain
    p = Problem(name=f"paper_burgers_{N}", pde=BURGERS, bc=DIRICHLET, nx=N, ny=N, nt=nt,
                x0=x0, x1=x1, y0=y0, y1=y1, dt=T / nt, m0=mu, m2=0.0)
    fn = lambda x, y, t: burgers_exact(x, y, t, mu, v)
    X, Y = p.grid()
    p.u0 = np.ascontiguousarray(fn(X, Y, 0.0).reshape(-1))
    p.ring = ring_from(p, fn)
    p.exact = fn
    return p


def exact_field(p: Problem, fn) -> np.ndarray:
    """fn at the unknown nodes of levels n = 1..nt, shape (nt, ns)."""
    X, Y = p.grid()
    return np.stack([fn(X, Y, n * p.dt).reshape(-1) for n in range(1, p.nt + 1)])


def custom(name, pde, bc, nx, ny, nt, dt, m0, m2, u0, ring=None, domain=(0.0, 1.0, 0.0, 1.0),
           newton_tol=1e-12) -> Problem:
    x0, x1, y0, y1 = domain
    p = Problem(name=name, pde=pde, bc=bc, nx=nx, ny=ny, nt=nt, x0=x0, x1=x1, y0=y0, y1=y1,
                dt=dt, m0=m0, m2=m2, newton_tol=newton_tol)
    p.u0 = np.ascontiguousarray(np.asarray(u0, dtype=np.float64).reshape(-1))
    assert p.u0.size == p.ns
    p.ring = None if ring is None else np.ascontiguousarray(np.asarray(ring, dtype=np.float64).reshape(nt, -1))
    return p
