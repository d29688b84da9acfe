"""Python face of the CPU ORACLE (ctypes over ``liboracle.so`` built from ``pit_oracle.c``).

TEST INFRASTRUCTURE ONLY: imported by ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
cpu_baseline / ``--impl reference`` leg, never by the product package.  It does not import the product
package either: problems are duck-typed (any object with the fields of the paper's problem statement:
pde, bc, nx, ny, nt, x0, x1, y0, y1, dt, m0, m2, u0, ring).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "pit_oracle.c")
LIB = os.path.join(HERE, "liboracle.so")


class OrProb(C.Structure):
    _fields_ = [("pde", C.c_int), ("bc", C.c_int), ("nx", C.c_int), ("ny", C.c_int), ("nt", C.c_int),
                ("x0", C.c_double), ("x1", C.c_double), ("y0", C.c_double), ("y1", C.c_double),
                ("dt", C.c_double), ("m0", C.c_double), ("m2", C.c_double)]


def build(force: bool = False) -> str:
    """Compile the oracle (plain C99, -O2, IEEE semantics: no -ffast-math)."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        tmp = LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-fPIC", "-shared", "-fno-fast-math",
                               "-o", tmp, SRC, "-lm"])
        os.replace(tmp, LIB)
    return LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(LIB)
        dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
        P = C.POINTER(OrProb)
        L.or_ns.argtypes = [P]; L.or_ns.restype = C.c_long
        L.or_residual.argtypes = [P, dp, dp, C.c_void_p, dp]; L.or_residual.restype = None
        L.or_jacobian.argtypes = [P, dp, C.c_void_p, dp, dp, dp, dp, dp]; L.or_jacobian.restype = None
        L.or_matvec.argtypes = [P, dp, dp, dp, dp, dp, dp, dp]; L.or_matvec.restype = None
        L.or_band_lu_solve.argtypes = [P, dp, dp, dp, dp, dp, dp, dp]; L.or_band_lu_solve.restype = C.c_int
        L.or_bicgstab_solve.argtypes = [P, dp, dp, dp, dp, dp, dp, dp, C.c_double, C.c_int]
        L.or_bicgstab_solve.restype = C.c_int
        L.or_solve_sequential.argtypes = [P, dp, C.c_void_p, C.c_int, dp, C.c_void_p, C.c_void_p]
        L.or_solve_sequential.restype = C.c_int
        L.or_solve_allatonce.argtypes = [P, dp, C.c_void_p, C.c_void_p, C.c_double, C.c_int, dp, dp,
                                         C.POINTER(C.c_int)]
        L.or_solve_allatonce.restype = C.c_int
        L.or_allatonce_iteration.argtypes = [P, dp, C.c_void_p, C.c_void_p, dp, dp, C.c_void_p, dp]
        L.or_allatonce_iteration.restype = C.c_int
        L.or_spacetime_residual.argtypes = [P, dp, C.c_void_p, dp, dp]
        L.or_spacetime_residual.restype = None
        _lib = L
    return _lib


def _prob(p) -> OrProb:
    return OrProb(int(p.pde), int(p.bc), int(p.nx), int(p.ny), int(p.nt), float(p.x0), float(p.x1),
                  float(p.y0), float(p.y1), float(p.dt), float(p.m0), float(p.m2))


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _ring_level(p, n):
    """Ring of level n (1-based) or None."""
    if p.bc != 0 or p.ring is None:
        return None
    return np.ascontiguousarray(p.ring[n - 1], dtype=np.float64)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def residual(p, u, uprev, n=1) -> np.ndarray:
    """G^n(u; uprev) (Eq. (3) times tau); the Newton rhs of Eq. (5) is -G."""
    pr = _prob(p)
    G = np.empty(lib().or_ns(C.byref(pr)))
    ring = _ring_level(p, n)
    lib().or_residual(C.byref(pr), _f64(u), _f64(uprev), _ptr(ring), G)
    return G


def jacobian(p, u, n=1):
    """(C, E, W, N, S) coefficient arrays of A_n = I + tau dF/du (Eq. (6))."""
    pr = _prob(p)
    ns = lib().or_ns(C.byref(pr))
    out = [np.empty(ns) for _ in range(5)]
    ring = _ring_level(p, n)
    lib().or_jacobian(C.byref(pr), _f64(u), _ptr(ring), *out)
    return tuple(out)


def matvec(p, coefs, x) -> np.ndarray:
    pr = _prob(p)
    y = np.empty_like(_f64(x))
    lib().or_matvec(C.byref(pr), *[_f64(c) for c in coefs], _f64(x), y)
    return y


def band_lu_solve(p, coefs, b) -> np.ndarray:
    pr = _prob(p)
    x = np.empty_like(_f64(b))
    rc = lib().or_band_lu_solve(C.byref(pr), *[_f64(c) for c in coefs], _f64(b), x)
    if rc != 0:
        raise RuntimeError(f"or_band_lu_solve rc={rc}")
    return x


def bicgstab_solve(p, coefs, b, rtol=1e-15, maxit=4000) -> np.ndarray:
    pr = _prob(p)
    x = np.empty_like(_f64(b))
    rc = lib().or_bicgstab_solve(C.byref(pr), *[_f64(c) for c in coefs], _f64(b), x, rtol, maxit)
    if rc < 0:
        raise RuntimeError(f"or_bicgstab_solve rc={rc}")
    return x


def to_dense(p, coefs) -> np.ndarray:
    """Assemble the 5-coefficient operator as a dense matrix by applying it to unit vectors."""
    ns = coefs[0].size
    A = np.empty((ns, ns))
    e = np.zeros(ns)
    for k in range(ns):
        e[k] = 1.0
        A[:, k] = matvec(p, coefs, e)
        e[k] = 0.0
    return A


class SeqResult:
    def __init__(self, U, iters, last_delta, status, seconds):
        self.U, self.iters, self.last_delta, self.status, self.seconds = U, iters, last_delta, status, seconds


def solve_sequential(p, levels=None) -> SeqResult:
    """Sequential BDF1 + Newton per level.  ``levels`` < nt solves a prefix (the
    system is block lower triangular in time, Eq. (6), so a prefix is exact)."""
    pr = _prob(p)
    ns = lib().or_ns(C.byref(pr))
    levels = p.nt if levels is None else levels
    U = np.empty(levels * ns)
    iters = np.zeros(levels, dtype=np.int32)
    last = np.zeros(levels)
    ring = None if (p.bc != 0 or p.ring is None) else _f64(p.ring)
    t0 = time.perf_counter()
    rc = lib().or_solve_sequential(C.byref(pr), _f64(p.u0), _ptr(ring), levels, U,
                                   iters.ctypes.data_as(C.c_void_p), last.ctypes.data_as(C.c_void_p))
    dt = time.perf_counter() - t0
    if rc not in (0, -4):
        raise RuntimeError(f"or_solve_sequential rc={rc}")
    return SeqResult(U.reshape(levels, ns), iters, last, rc, dt)


class AaoResult:
    def __init__(self, U, hist, niter, status):
        self.U, self.hist, self.niter, self.status = U, hist, niter, status


def solve_allatonce(p, tol=None, newton_max=30, guess=None) -> AaoResult:
    """Test-only global Newton (Eq. (5)-(7)) with the GPU's initial guess and stop rule."""
    pr = _prob(p)
    ns = lib().or_ns(C.byref(pr))
    tol = p.newton_tol if tol is None else tol
    U = np.empty(p.nt * ns)
    hist = np.zeros(4 * newton_max)
    nit = C.c_int(0)
    ring = None if (p.bc != 0 or p.ring is None) else _f64(p.ring)
    g = None if guess is None else _f64(guess)
    rc = lib().or_solve_allatonce(C.byref(pr), _f64(p.u0), _ptr(ring), _ptr(g), tol, newton_max, U, hist,
                                  C.byref(nit))
    if rc < -1 and rc != -4:
        raise RuntimeError(f"or_solve_allatonce rc={rc}")
    return AaoResult(U.reshape(p.nt, ns), hist.reshape(newton_max, 4)[: nit.value], nit.value, rc)


def spacetime_residual(p, U) -> np.ndarray:
    """R = -G^n(U^n; U^{n-1}) for all levels (shape (nt, ns))."""
    pr = _prob(p)
    ns = lib().or_ns(C.byref(pr))
    R = np.empty(p.nt * ns)
    ring = None if (p.bc != 0 or p.ring is None) else _f64(p.ring)
    lib().or_spacetime_residual(C.byref(pr), _f64(p.u0), _ptr(ring), _f64(np.asarray(U).reshape(-1)), R)
    return R.reshape(p.nt, ns)


def allatonce_iteration(p, u_prev, carry_in, Uk):
    """ONE all-at-once Newton iteration over a slab (levels 1..p.nt after the level u_prev, incoming carry
    carry_in or None = 0): returns (U_{k+1}, carry_out, sums {sum R^2, max|R|, sum dU^2, max|dU|})."""
    pr = _prob(p)
    ns = lib().or_ns(C.byref(pr))
    Uk1 = np.empty(p.nt * ns)
    cout = np.empty(ns)
    sums = np.zeros(4)
    ring = None if (p.bc != 0 or p.ring is None) else _f64(p.ring)
    ci = None if carry_in is None else _f64(carry_in)
    rc = lib().or_allatonce_iteration(C.byref(pr), _f64(u_prev), _ptr(ci), _ptr(ring), _f64(np.asarray(Uk).reshape(-1)),
                                      Uk1, cout.ctypes.data_as(C.c_void_p), sums)
    if rc != 0:
        raise RuntimeError(f"or_allatonce_iteration rc={rc}")
    return Uk1.reshape(p.nt, ns), cout, sums
