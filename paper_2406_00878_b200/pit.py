"""Thin ctypes binding of libpit (include/pit.h) — argument marshalling only.

Every step of the hot path runs in libpit's CUDA kernels; this module only converts arguments.  PyTorch
is used for device memory and streams (``tensor.data_ptr()``, ``torch.cuda.current_stream()``).  There is
no fallback: if ``libpit.so`` is missing or no sm_100 device is usable, calls raise.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional

import numpy as np

from . import workloads as W

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libpit.so")

PIT_ABI_VERSION = 3
PIT_OK, PIT_OK_FLOOR, PIT_EINVAL, PIT_ENOMEM, PIT_ECUDA, PIT_ENOCONV, PIT_EBREAKDOWN, PIT_ECOND = 0, 1, -1, -2, -3, -4, -5, -6
PIT_HEAT, PIT_BURGERS = 0, 1
PIT_DIRICHLET, PIT_PERIODIC = 0, 1
PIT_INV_AUTO, PIT_INV_RECURRENCE, PIT_INV_PRODUCT_WINDOW, PIT_INV_EXPLICIT = 0, 1, 2, 3

# every symbol include/pit.h declares (tests check the library exports all of them)
EXPORTS = ["pit_config_init", "pit_create", "pit_workspace_bytes", "pit_create_with_workspace", "pit_destroy", "pit_solve", "pit_solve_device", "pit_residual_device",
           "pit_level_solve_device", "pit_product_window_device", "pit_slab_iterate_device", "pit_explicit_window_device", "pit_initial_guess_device", "pit_sizes", "pit_stats", "pit_engine_info", "pit_strerror",
           "pit_last_error", "pit_abi_version"]


class PitConfig(C.Structure):
    _fields_ = [("abi_version", C.c_int32), ("pde", C.c_int32), ("bc", C.c_int32), ("nx", C.c_int32),
                ("ny", C.c_int32), ("nt", C.c_int32), ("x0", C.c_double), ("x1", C.c_double), ("y0", C.c_double),
                ("y1", C.c_double), ("dt", C.c_double), ("m0", C.c_double), ("m2", C.c_double),
                ("newton_tol", C.c_double), ("newton_max", C.c_int32), ("lin_rtol", C.c_double),
                ("lin_atol", C.c_double), ("lin_max", C.c_int32), ("inverse_mode", C.c_int32),
                ("window", C.c_int32), ("pipeline_depth", C.c_int32), ("device", C.c_int32),
                ("engine", C.c_int32), ("guess_cf", C.c_int32), ("stop_norm", C.c_int32),
                ("lin_sweeps", C.c_int32), ("lin_check", C.c_int32)]


class PitError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"libpit error {code}: {msg}")
        self.code = code


_lib = None


def lib():
    """Load libpit.so (raises if it was not built: there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} not built: run `python -m paper_2406_00878_b200.build`")
        L = C.CDLL(LIB_PATH)
        vp, dp, i32p, hp = C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p
        L.pit_config_init.argtypes = [C.POINTER(PitConfig)]; L.pit_config_init.restype = None
        L.pit_create.argtypes = [C.POINTER(PitConfig), C.POINTER(C.c_void_p)]; L.pit_create.restype = C.c_int
        L.pit_destroy.argtypes = [hp]; L.pit_destroy.restype = None
        L.pit_workspace_bytes.argtypes = [C.POINTER(PitConfig), C.POINTER(C.c_size_t)]
        L.pit_workspace_bytes.restype = C.c_int
        L.pit_create_with_workspace.argtypes = [C.POINTER(PitConfig), vp, C.c_size_t, C.POINTER(C.c_void_p)]
        L.pit_create_with_workspace.restype = C.c_int
        L.pit_solve.argtypes = [hp, dp, dp, dp, dp, dp, i32p]; L.pit_solve.restype = C.c_int
        L.pit_solve_device.argtypes = [hp, dp, dp, dp, dp, dp, i32p, vp]; L.pit_solve_device.restype = C.c_int
        L.pit_residual_device.argtypes = [hp, dp, dp, dp, dp, dp, dp, vp]; L.pit_residual_device.restype = C.c_int
        L.pit_level_solve_device.argtypes = [hp, C.c_int32, dp, dp, dp, dp, i32p, vp]
        L.pit_level_solve_device.restype = C.c_int
        L.pit_product_window_device.argtypes = [hp, C.c_int32, C.c_int32, dp, dp, dp, dp, dp, dp, i32p, vp]
        L.pit_product_window_device.restype = C.c_int
        L.pit_explicit_window_device.argtypes = [hp, C.c_int32, C.c_int32, dp, dp, dp, dp, dp, dp, i32p, vp]
        L.pit_explicit_window_device.restype = C.c_int
        L.pit_initial_guess_device.argtypes = [hp, dp, dp, dp, vp]; L.pit_initial_guess_device.restype = C.c_int
        L.pit_slab_iterate_device.argtypes = [hp, dp, dp, dp, dp, dp, dp, dp, i32p, vp]
        L.pit_slab_iterate_device.restype = C.c_int
        L.pit_sizes.argtypes = [hp, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]; L.pit_sizes.restype = C.c_int
        L.pit_stats.argtypes = [hp, C.POINTER(C.c_int64), C.c_int32]; L.pit_stats.restype = C.c_int
        L.pit_engine_info.argtypes = [hp, C.POINTER(C.c_double), C.c_int32]; L.pit_engine_info.restype = C.c_int
        L.pit_strerror.argtypes = [C.c_int]; L.pit_strerror.restype = C.c_char_p
        L.pit_last_error.argtypes = [hp]; L.pit_last_error.restype = C.c_char_p
        L.pit_abi_version.argtypes = []; L.pit_abi_version.restype = C.c_int
        _lib = L
    return _lib


def make_config(p: W.Problem, **over) -> PitConfig:
    c = PitConfig()
    lib().pit_config_init(C.byref(c))
    c.pde, c.bc, c.nx, c.ny, c.nt = p.pde, p.bc, p.nx, p.ny, p.nt
    c.x0, c.x1, c.y0, c.y1 = p.x0, p.x1, p.y0, p.y1
    c.dt, c.m0, c.m2, c.newton_tol = p.dt, p.m0, p.m2, p.newton_tol
    for k, v in over.items():
        setattr(c, k, v)
    return c


def _ptr(t) -> Optional[int]:
    if t is None:
        return None
    if isinstance(t, np.ndarray):
        assert t.dtype == np.float64 and t.flags.c_contiguous
        return t.ctypes.data
    assert t.is_contiguous(), "tensor must be contiguous"
    return t.data_ptr()


def _stream(stream) -> Optional[int]:
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    return getattr(stream, "cuda_stream", stream)


def workspace_bytes(p: W.Problem, **cfg_over) -> int:
    """pit_workspace_bytes: the device bytes a handle for problem ``p`` holds."""
    cfg = make_config(p, **cfg_over)
    n = C.c_size_t(0)
    rc = lib().pit_workspace_bytes(C.byref(cfg), C.byref(n))
    if rc != 0:
        raise PitError(rc, lib().pit_strerror(rc).decode())
    return int(n.value)


class Solver:
    """One libpit handle for one problem shape (pit_create / pit_destroy).  ``workspace``: a device buffer (a torch
    tensor of >= workspace_bytes(p) bytes) the handle carves its memory from (pit_create_with_workspace); the
    Solver keeps a reference to it."""

    def __init__(self, p: W.Problem, workspace=None, **cfg_over):
        self.problem = p
        self.cfg = make_config(p, **cfg_over)
        self.workspace = workspace
        h = C.c_void_p()
        if workspace is None:
            rc = lib().pit_create(C.byref(self.cfg), C.byref(h))
        else:
            nbytes = workspace.numel() * workspace.element_size()
            rc = lib().pit_create_with_workspace(C.byref(self.cfg), C.c_void_p(workspace.data_ptr()), nbytes, C.byref(h))
        if rc != 0:
            raise PitError(rc, lib().pit_strerror(rc).decode())
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            try:
                lib().pit_destroy(self.h)
            except TypeError:          # interpreter shutdown: module globals already torn down
                pass
            self.h = None

    __del__ = close

    def _check(self, rc):
        if rc < 0 and rc not in (PIT_ENOCONV, PIT_EBREAKDOWN):
            raise PitError(rc, lib().pit_last_error(self.h).decode())
        return rc

    # -- host path (pit_solve) --
    def solve_host(self, u0: np.ndarray, ring=None, guess=None):
        p = self.problem
        u_out = np.empty((p.nt, p.ns))
        hist = np.zeros((self.cfg.newton_max, 4))
        nit = C.c_int32(0)
        rc = lib().pit_solve(self.h, _ptr(np.ascontiguousarray(u0, dtype=np.float64)),
                             None if ring is None else _ptr(np.ascontiguousarray(ring, dtype=np.float64)),
                             None if guess is None else _ptr(np.ascontiguousarray(guess, dtype=np.float64)),
                             _ptr(u_out), _ptr(hist), C.addressof(nit))
        self._check(rc)
        return u_out, hist[: nit.value], nit.value, rc

    # -- device path (pit_solve_device) --
    def solve_device(self, d_u0, d_ring, d_guess, d_out, d_hist, d_info, stream=None) -> int:
        return self._check(lib().pit_solve_device(self.h, _ptr(d_u0), _ptr(d_ring), _ptr(d_guess), _ptr(d_out),
                                                  _ptr(d_hist), _ptr(d_info), _stream(stream)))

    def residual_device(self, d_U, d_u0, d_ring, d_R, d_diag=None, d_norms=None, stream=None) -> int:
        return self._check(lib().pit_residual_device(self.h, _ptr(d_U), _ptr(d_u0), _ptr(d_ring), _ptr(d_R),
                                                     _ptr(d_diag), _ptr(d_norms), _stream(stream)))

    def initial_guess_device(self, d_u0, d_ring, d_U0, stream=None) -> int:
        return self._check(lib().pit_initial_guess_device(self.h, _ptr(d_u0), _ptr(d_ring), _ptr(d_U0), _stream(stream)))

    def slab_iterate_device(self, d_uprev, d_carry_in, d_ring, d_U_k, d_U_k1, d_carry_out, d_hist, d_info=None,
                            stream=None) -> int:
        return self._check(lib().pit_slab_iterate_device(self.h, _ptr(d_uprev), _ptr(d_carry_in), _ptr(d_ring),
                                                         _ptr(d_U_k), _ptr(d_U_k1), _ptr(d_carry_out), _ptr(d_hist),
                                                         _ptr(d_info), _stream(stream)))

    def level_solve_device(self, level, d_U, d_ring, d_b, d_x, d_info, stream=None) -> int:
        return self._check(lib().pit_level_solve_device(self.h, level, _ptr(d_U), _ptr(d_ring), _ptr(d_b),
                                                        _ptr(d_x), _ptr(d_info), _stream(stream)))

    def product_window_device(self, s0, L, d_U, d_u0, d_ring, d_R, d_carry, d_dU, d_info, stream=None) -> int:
        return self._check(lib().pit_product_window_device(self.h, s0, L, _ptr(d_U), _ptr(d_u0), _ptr(d_ring),
                                                           _ptr(d_R), _ptr(d_carry), _ptr(d_dU), _ptr(d_info),
                                                           _stream(stream)))

    def explicit_window_device(self, s0, L, d_U, d_u0, d_ring, d_R, d_carry, d_dU, d_info, stream=None) -> int:
        return self._check(lib().pit_explicit_window_device(self.h, s0, L, _ptr(d_U), _ptr(d_u0), _ptr(d_ring),
                                                            _ptr(d_R), _ptr(d_carry), _ptr(d_dU), _ptr(d_info),
                                                            _stream(stream)))

    def stats(self):
        out = (C.c_int64 * (17 + 256 + 8))()
        self._check(lib().pit_stats(self.h, out, 17 + 256 + 8))
        d = {"steps": out[0], "inner_iterations": out[1], "depth": out[2], "grid": out[3], "launches": out[4],
             "newton_kernel_ms": out[5] * 1e-6, "init_kernel_ms": out[6] * 1e-6, "engine": out[7],
             "product_form": bool(out[15]), "explicit_form": out[15] == 2, "pair_iterations": out[16],
             "iterations_per_newton_k": [out[17 + k] for k in range(256) if out[17 + k]],
             "guess_ms": out[279] * 1e-6, "grid_barriers": out[280]}
        if any(out[8:15]):
            names = ["prologue", "phase1", "phase2", "epilogue", "barrier", "reduce", "step_tail"]
            d["trace_cycles_per_cta"] = {k: out[8 + i] / max(1, out[3]) for i, k in enumerate(names)}
            sub = ["pro_loads", "pro_wait", "pro_residual", "pro_x0mv", "step_setup", "pro_stage"]
            d["trace_cycles_per_cta"].update({k: out[273 + i] / max(1, out[3]) for i, k in enumerate(sub)})
        return d

    def engine_info(self):
        """pit_engine_info: engine, omega, sweeps, Jacobi bound and per-iteration level-solve residuals."""
        n = 4 + 2 * 256 + 16
        out = (C.c_double * n)()
        self._check(lib().pit_engine_info(self.h, out, n))
        lr = [(out[4 + 2 * k], out[5 + 2 * k]) for k in range(256)]
        while lr and lr[-1] == (0.0, 0.0):
            lr.pop()
        d = {"engine": int(out[0]), "omega": out[1], "sweeps": int(out[2]), "q": out[3], "linres": lr}
        b = 4 + 2 * 256
        if any(out[b:b + 16]):
            names = ["prologue", "sweeps", "sweep_waits", "epilogue", "reductions", "pass_ends", "step_setup", "total"]
            d["trace_mean"] = {k: out[b + i] for i, k in enumerate(names)}
            d["trace_max"] = {k: out[b + 8 + i] for i, k in enumerate(names)}
        return d

    def sizes(self):
        ns, b = C.c_int64(), C.c_int64()
        self._check(lib().pit_sizes(self.h, C.byref(ns), C.byref(b)))
        return ns.value, b.value


def solve(p: W.Problem, device=True, **cfg_over):
    """Convenience: solve problem ``p`` on the GPU; returns (U [nt, ns] numpy, hist, n_iter, status)."""
    s = Solver(p, **cfg_over)
    try:
        return s.solve_host(p.u0, p.ring)
    finally:
        s.close()
