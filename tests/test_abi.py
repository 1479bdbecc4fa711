"""The C-ABI library loads without a GPU and exports every symbol declared in
include/*.h; the product never imports the oracle."""
import ctypes as C
import glob
import os
import re

from paper_2006_02602_b200 import capi

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


def declared_functions():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        src = open(h).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        for m in re.finditer(r"^[A-Za-z_][\w\s\*]*?\b(cav_\w+)\s*\(", src, flags=re.M):
            names.add(m.group(1))
    return sorted(names)


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("cav_residual_box", "cav_update_box", "cav_run_case", "cav_block_create",
                 "cav_block_run", "cav_block_connect", "cav_block_arena_ipc", "cav_last_error"):
        assert must in names


def test_library_exports_every_declared_symbol():
    for fmad in (False, True):
        L = C.CDLL(capi.lib_path(fmad))
        missing = [n for n in declared_functions() if not hasattr(L, n)]
        assert not missing, (fmad, missing)


def test_version_and_error_channel():
    assert "sm_100a" in capi.version() and "fmad=false" in capi.version()
    assert "fmad=true" in capi.version(True)
    try:
        capi.choose_dims(0, "3d")
    except capi.InvalidArgument as e:
        assert str(e) == "choose_dims: np must be >= 1"
    else:
        raise AssertionError("expected InvalidArgument")


def test_product_does_not_import_the_oracle():
    pkg = os.path.join(ROOT, "paper_2006_02602_b200")
    banned = re.compile(r"(from\s+oracle|import\s+oracle|refbind|libcavity_oracle|libcavity_ref|"
                        r"cavity_oracle\.h)")
    for path in glob.glob(os.path.join(pkg, "**", "*.*"), recursive=True):
        if path.endswith((".py", ".cu", ".cuh", ".cpp", ".hpp")):
            assert not banned.search(open(path).read()), path


def test_sm100a_cubin_in_library():
    data = open(capi.lib_path(), "rb").read()
    assert b"sm_100a" in data or b"sm_100" in data


def test_cpp_header_rethrows_reference_exceptions(tmp_path):
    """include/cavity_b200.hpp maps status codes back onto the reference's
    exception types and messages (compiled and run here, host logic only)."""
    import shutil
    import subprocess
    if not shutil.which("g++"):
        return
    src = tmp_path / "t.cpp"
    src.write_text(r'''
#include <cstdio>
#include "cavity_b200.hpp"
int main() {
  int d[3];
  try { cavity_b200::check(cav_choose_dims(7, CAV_MODE_2D, d)); return 1; }
  catch (const std::invalid_argument& e) { std::printf("%s\n", e.what()); }
  cavity_b200::check(cav_choose_dims(8, CAV_MODE_3D, d));
  std::printf("%d %d %d\n", d[0], d[1], d[2]);
  return 0;
}''')
    exe = tmp_path / "t"
    lib_dir = os.path.dirname(capi.lib_path())
    subprocess.run(["g++", "-std=c++17", "-I", os.path.join(ROOT, "include"), str(src), "-L", lib_dir,
                    "-lcavity_b200", f"-Wl,-rpath,{lib_dir}", "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.splitlines()
    assert out[0].startswith("choose_dims: 2d cannot split a prime rank count 7")
    assert out[1] == "2 2 2"


def test_ctypes_prototypes_match_header():
    """Every argtypes list capi.py declares has the arity of the header's
    prototype (a stale list turns a call into a TypeError on the GPU box)."""
    import re
    from paper_2006_02602_b200 import capi
    src = open(os.path.join(ROOT, "include", "cavity_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    protos = {}
    for m in re.finditer(r"\b(?:int|void|double|const char\*)\s+(cav_\w+)\s*\(([^;{]*?)\)\s*;", src, flags=re.S):
        args = m.group(2).strip()
        depth, n = 0, (0 if args in ("", "void") else 1)
        for ch in args:
            depth += ch in "([" and 1 or 0
            depth -= ch in ")]" and 1 or 0
            n += ch == "," and depth == 0
        protos[m.group(1)] = n
    L = capi.lib()
    checked = 0
    for name, n in protos.items():
        at = getattr(getattr(L, name), "argtypes", None)
        if at is not None:
            assert len(at) == n, (name, len(at), n)
            checked += 1
    assert checked >= 10


def test_integration_driver_seam_compiles_against_the_reference(tmp_path):
    """INTEGRATION.md §2's run_case_b200 (the reference-side binding a
    maintainer adds) compiles against the reference's own headers and ours
    (g++ -std=c++20 -fsyntax-only); skipped where the reference is absent."""
    import shutil
    import subprocess
    import pytest
    ref_inc = "/root/reference/proj/include"
    if not os.path.isdir(ref_inc) or not shutil.which("g++"):
        pytest.skip("reference headers not available")
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    blocks = re.findall(r"```cpp\n(.*?)```", text, flags=re.S)
    seam = [b for b in blocks if "run_case_b200" in b]
    assert seam, "INTEGRATION.md lost its run_case seam"
    src = tmp_path / "seam.cpp"
    src.write_text('#include "cavity_b200.h"\n#include <cstring>\n#include <stdexcept>\n#include <vector>\n#include <algorithm>\n'
                   '#include "cavity/runner.hpp"\n#include "cavity/transport.hpp"\n'
                   'namespace cavity {\n' + seam[0] + '\n}\n')
    p = subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-Wno-return-type", "-I", ref_inc, "-I",
                        os.path.join(ROOT, "include"), str(src)], capture_output=True, text=True)
    assert p.returncode == 0, p.stderr[-3000:]
