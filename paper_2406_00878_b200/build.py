"""Build libpit.so in-tree for sm_100a (nvcc cross-compiles without a GPU).

Five translation units compiled in parallel and linked into one shared library: pit_api.cu (the C ABI, engines
1-3, kernel (a), the product forms, the coarse guess) and the engine-4 instantiations pit_nb_law0.cu /
pit_nb_law1.cu (pit_newton_nb.cuh) and the engine-5 instantiations pit_ps_law1.cu (pit_newton_ps.cuh) and pit_ps_law0.cu (pit_newton_ps0.cuh).
"""
from __future__ import annotations

import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libpit.so")
UNITS = ["pit_api.cu", "pit_nb_law1.cu", "pit_nb_law0.cu", "pit_ps_law1.cu", "pit_ps_law0.cu"]
SOURCES = UNITS + ["pit_kernels.cu", "pit_internal.cuh", "pit_newton_onchip.cuh", "pit_newton_col.cuh",
                   "pit_guess.cuh", "pit_explicit.cuh", "pit_newton_nb.cuh", "pit_nb_params.cuh", "pit_newton_ps.cuh", "pit_newton_ps0.cuh", "pit_ps_params.cuh"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v"]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, s) for s in SOURCES] + [os.path.join(ROOT, "include", "pit.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    tag = f"tmp{os.getpid()}"
    objs, procs = [], []
    for u in UNITS:
        o = os.path.join(CSRC, u.replace(".cu", f".{tag}.o"))
        objs.append(o)
        cmd = [nvcc, *NVCC_FLAGS, "-I", os.path.join(ROOT, "include"), "-c", "-o", o, os.path.join(CSRC, u)]
        procs.append(subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True))
    logs, failed = [], []
    for u, pr in zip(UNITS, procs):
        out, err = pr.communicate()
        logs.append(err)
        if pr.returncode != 0:
            failed.append(f"{u}:\n{err}")
    try:
        if failed:
            raise RuntimeError("nvcc failed:\n" + "\n".join(failed))
        tmp = LIB + f".{tag}"
        link = subprocess.run([nvcc, *ARCH, "-shared", "-o", tmp, *objs, "-ldl"], capture_output=True, text=True)
        if link.returncode != 0:
            raise RuntimeError(f"link failed:\n{link.stderr}")
        os.replace(tmp, LIB)
    finally:
        for o in objs:
            if os.path.exists(o):
                os.remove(o)
    if verbose:
        print("\n".join(logs))
    return LIB


if __name__ == "__main__":
    print(build(force=True, verbose=True))
