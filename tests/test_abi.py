"""The C-ABI library loads on a CPU-only box and exports every symbol include/cr.h declares;
the Python binding wraps each of them (no compute calls: no GPU here)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "cr.h")
LIB = os.path.join(ROOT, "paper_2101_03777_b200", "libcr.so")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(cr_[a-z_0-9]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(LIB):
        import importlib.util
        spec = importlib.util.spec_from_file_location("_cr_build", os.path.join(ROOT, "paper_2101_03777_b200", "build.py"))
        b = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(b)
        b.build()
    return ctypes.CDLL(LIB)


def test_header_declares_the_north_star_calls():
    syms = declared_symbols()
    for s in ("cr_build_mesh", "cr_assemble_coupled", "cr_hybridise", "cr_solve", "cr_recover"):
        assert s in syms


def test_library_exports_every_declared_symbol(lib):
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_binding_wraps_every_symbol(lib):
    import paper_2101_03777_b200 as P
    assert sorted(P.ABI_SYMBOLS) == declared_symbols()
    lib.cr_version.restype = ctypes.c_char_p
    assert b"sm_100a" in lib.cr_version()


def test_invalid_arguments_fail_cleanly_without_gpu(lib):
    # argument validation happens before any CUDA call
    lib.cr_build_mesh.restype = ctypes.c_int
    lib.cr_last_error.restype = ctypes.c_char_p
    out = ctypes.c_void_p()
    st = lib.cr_build_mesh(ctypes.c_int32(4), ctypes.c_int64(3), None, ctypes.c_int64(1), None, None,
                           ctypes.byref(out))
    assert st == -1 and b"dim" in lib.cr_last_error()
    assert out.value is None


def test_new_entry_points_validate_arguments_without_gpu(lib):
    lib.cr_last_error.restype = ctypes.c_char_p
    lib.cr_newton_update.restype = ctypes.c_int
    assert lib.cr_newton_update(ctypes.c_int64(-1), None, None, ctypes.c_int64(0), None, None, ctypes.c_double(1.0),
                                None, None) == -1
    lib.cr_coupled_rhs_norm.restype = ctypes.c_int
    assert lib.cr_coupled_rhs_norm(None, None, None, None, None) == -1
    lib.cr_hybrid_method_host.restype = ctypes.c_int
    assert lib.cr_hybrid_method_host(ctypes.c_int32(2), ctypes.c_int64(3), None, ctypes.c_int64(1), None,
                                     None, None, None, None, None, None, None, None, None, None) == -1
    assert b"null" in lib.cr_last_error()
    lib.cr_pool_reserve.restype = ctypes.c_int
    assert lib.cr_pool_reserve(ctypes.c_int64(-5), None) == -1
    lib.cr_kernel_launches.restype = ctypes.c_int64
    assert lib.cr_kernel_launches() == 0          # nothing launched on a CPU box


def test_struct_layouts_match_the_header(tmp_path):
    """sizeof / offsetof of the ABI structs as gcc lays them out from include/cr.h equal the
    ctypes mirrors of the binding (a mismatch would silently shift every later field)."""
    import shutil
    import subprocess
    import paper_2101_03777_b200 as P
    if not shutil.which("gcc"):
        pytest.skip("gcc not available")
    structs = {"cr_solver_opts": P.SolverOpts, "cr_solve_report": P.SolveReport, "cr_params": P.Params,
               "cr_data": P.Data, "cr_mesh_info_t": P.MeshInfo}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "cr.h"', 'int main(void) {']
    for cname, py in structs.items():
        lines.append(f'printf("{cname} %zu\\n", sizeof({cname}));')
        for f, _ in py._fields_:
            lines.append(f'printf("{cname}.{f} %zu\\n", offsetof({cname}, {f}));')
    lines.append("return 0; }")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    got = dict(l.split() for l in subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split("\n") if l)
    for cname, py in structs.items():
        assert int(got[cname]) == ctypes.sizeof(py), cname
        for f, _ in py._fields_:
            assert int(got[f"{cname}.{f}"]) == getattr(py, f).offset, (cname, f)
