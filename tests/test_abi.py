"""The C-ABI library loads and exports every entry point include/castfem_b200.h declares
(no GPU needed: no compute call is made)."""
import ctypes as C
import os
import re

from paper_1005_3158_b200 import _abi

HDR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "castfem_b200.h")


def declared():
    src = open(HDR).read()
    return sorted(set(re.findall(r"^int\s+(cf_\w+)\s*\(", src, re.M)))


def test_header_declares_entry_points():
    names = declared()
    assert "cf_plan_create" in names and "cf_step" in names and len(names) >= 25


def test_library_exports_every_declared_symbol():
    lib = _abi.lib()
    for name in declared():
        assert hasattr(lib, name), name


def test_python_mirror_binds_every_declared_symbol():
    bound = {n for n, _, _ in _abi.SIGNATURES}
    assert set(declared()) <= bound


def test_abi_version_and_error_buffer():
    lib = _abi.lib()
    assert lib.cf_abi_version() == 2
    buf = C.create_string_buffer(64)
    assert lib.cf_last_error(buf, 64) == 0
    assert lib.cf_last_error(None, 0) == _abi.CF_INVALID_ARG


def test_library_is_sm100a_only():
    out = os.popen(f"cuobjdump --list-elf {_abi.LIB_PATH} 2>/dev/null").read()
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def test_cpp_shim_compiles_standalone(tmp_path):
    """include/castfem_b200.hpp compiles without the reference headers (templates over
    the caller's types) and links against the C-ABI library."""
    import subprocess
    src = tmp_path / "t.cpp"
    src.write_text('#include "castfem_b200.hpp"\nint main() { return cf_abi_version() == 2 ? 0 : 1; }\n')
    inc = os.path.join(os.path.dirname(HDR))
    libdir = os.path.dirname(_abi.LIB_PATH)
    r = subprocess.run(["g++", "-std=c++20", f"-I{inc}", str(src), "-o", str(tmp_path / "t"), f"-L{libdir}",
                        "-lcastfem_b200", f"-Wl,-rpath,{libdir}"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert subprocess.run([str(tmp_path / "t")]).returncode == 0


def test_c_header_is_plain_c(tmp_path):
    """The boundary is a C ABI: include/castfem_b200.h compiles as C11 (no C++ or torch types in
    any signature) and a C program links the library and calls through it."""
    import subprocess
    src = tmp_path / "t.c"
    src.write_text('#include "castfem_b200.h"\n#include <string.h>\n'
                   "int main(void) { char b[8]; cf_last_error(b, sizeof b); return cf_abi_version() == 2 ? 0 : 1; }\n")
    inc = os.path.join(os.path.dirname(HDR))
    libdir = os.path.dirname(_abi.LIB_PATH)
    r = subprocess.run(["gcc", "-std=c11", "-Wall", "-Werror", f"-I{inc}", str(src), "-o", str(tmp_path / "t"),
                        f"-L{libdir}", "-lcastfem_b200", f"-Wl,-rpath,{libdir}"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert subprocess.run([str(tmp_path / "t")]).returncode == 0
