"""CPU-side checks of the C-ABI boundary: libpit.so builds for sm_100a, loads, and exports every symbol
include/pit.h declares; argument validation works without a GPU (no compute calls here)."""
import ctypes as C
import os
import re
import shutil

import pytest

from paper_2406_00878_b200 import pit, workloads as W

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "pit.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pit_[a-z_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def built():
    if not os.path.exists(pit.LIB_PATH):
        if shutil.which("nvcc") is None and not os.path.exists("/usr/local/cuda/bin/nvcc"):
            pytest.skip("nvcc unavailable and libpit.so not built")
        from paper_2406_00878_b200 import build
        build.build()
    return pit.lib()


def test_header_and_binding_agree():
    assert _declared() == sorted(pit.EXPORTS)


def test_library_exports_every_declared_symbol(built):
    for name in _declared():
        assert hasattr(built, name), name
    assert built.pit_abi_version() == pit.PIT_ABI_VERSION


def test_config_struct_layout_matches_header(built, tmp_path):
    # offsets the C compiler sees: pit_config_init writes abi_version/newton_tol/newton_max at their C offsets
    c = pit.PitConfig()
    built.pit_config_init(C.byref(c))
    assert c.abi_version == pit.PIT_ABI_VERSION == 3 and c.newton_tol == 1e-12 and c.newton_max == 30 and c.x1 == 1.0 and c.y1 == 1.0
    assert c.pde == 0 and c.device == 0 and c.pipeline_depth == 0 and c.guess_cf == 0 and c.stop_norm == 0
    assert c.lin_sweeps == 0 and c.lin_check == 0
    # every field's offset and the struct size, as gcc lays out include/pit.h, against the ctypes binding
    if shutil.which("gcc") is None:
        pytest.skip("gcc unavailable")
    names = [f[0] for f in pit.PitConfig._fields_]
    prog = "#include <stdio.h>\n#include <stddef.h>\n#include \"pit.h\"\nint main(void){\n"
    prog += "".join(f'printf("%zu\\n", offsetof(pit_config, {n}));\n' for n in names)
    prog += 'printf("%zu\\n", sizeof(pit_config)); return 0; }\n'
    src = tmp_path / "layout.c"
    src.write_text(prog)
    exe = tmp_path / "layout"
    import subprocess
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), "-o", str(exe), str(src)])
    got = [int(v) for v in subprocess.check_output([str(exe)]).split()]
    assert got[:-1] == [getattr(pit.PitConfig, n).offset for n in names]
    assert got[-1] == C.sizeof(pit.PitConfig)


def test_strerror(built):
    assert built.pit_strerror(0) == b"converged"
    assert b"Newton" in built.pit_strerror(-4)


@pytest.mark.parametrize("field,value", [("abi_version", 7), ("nx", 1), ("nt", 0), ("dt", 0.0), ("m0", -1.0),
                                         ("newton_max", 0), ("pipeline_depth", 99), ("bc", 5),
                                         ("guess_cf", 1), ("guess_cf", 5), ("guess_cf", -2), ("stop_norm", 2),
                                         ("engine", 6), ("lin_sweeps", -1), ("lin_sweeps", 401), ("lin_check", -1)])
def test_invalid_config_rejected_before_touching_the_gpu(built, field, value):
    c = pit.make_config(W.config(1))
    setattr(c, field, value)
    h = C.c_void_p()
    assert built.pit_create(C.byref(c), C.byref(h)) == pit.PIT_EINVAL
    assert not h.value


def test_periodic_needs_three_intervals(built):
    c = pit.make_config(W.config(2, n=8, nt=2))
    c.nx = 2
    h = C.c_void_p()
    assert built.pit_create(C.byref(c), C.byref(h)) == pit.PIT_EINVAL


def test_null_handle_is_safe(built):
    built.pit_destroy(None)
    assert built.pit_solve(None, None, None, None, None, None, None) == pit.PIT_EINVAL
