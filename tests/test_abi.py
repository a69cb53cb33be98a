"""CPU-side checks of the C-ABI boundary: the library builds/loads and exports every symbol the
header declares; host logic that needs no GPU (argument validation paths are exercised on GPU)."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "cpqr.h")
LIB = os.path.join(ROOT, "paper_2112_10855_b200", "libcpqr.so")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(cpqr_[a-z_0-9]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(LIB):
        from paper_2112_10855_b200 import build
        build.build(verbose=False)
    return LIB


def test_header_declares_the_north_star_calls():
    names = declared_functions()
    for must in ["cpqr_create", "cpqr_set_tensor", "cpqr_set_factors", "cpqr_init_factors", "cpqr_sweep",
                 "cpqr_get_factors", "cpqr_get_fit", "cpqr_destroy"]:
        assert must in names


def test_library_exports_every_declared_symbol(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", lib], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\b(cpqr_[a-z_0-9]+)\b", out))
    missing = [n for n in declared_functions() if n not in exported]
    assert not missing, missing
    # nothing else leaks out of the library (hidden visibility)
    assert not [n for n in exported if n not in declared_functions()]


def test_binding_loads_and_matches_exports(lib):
    from paper_2112_10855_b200 import cpqr
    assert "sm_100a" in cpqr.version()
    assert sorted(cpqr.EXPORTS) == declared_functions()


def test_sass_is_sm100a_and_uses_dmma(lib):
    out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
    assert "sm_100a" in out
    assert "DMMA.8x8x4" in out  # FP64 tensor-core path of the Multi-TTM


def test_options_struct_layout_matches_binding(tmp_path):
    """The ctypes mirror of cpqr_options (and cpqr_profile) has the C header's size and offsets."""
    import ctypes as C
    from paper_2112_10855_b200 import cpqr
    fields = [f[0] for f in cpqr.Options._fields_]
    src = tmp_path / "lay.c"
    src.write_text('#include <stddef.h>\n#include <stdio.h>\n#include "cpqr.h"\nint main(void){\n'
                   + f'printf("%zu\\n", sizeof(cpqr_options));\n'
                   + "".join(f'printf("%zu\\n", offsetof(cpqr_options, {f}));\n' for f in fields)
                   + 'printf("%zu\\n", sizeof(cpqr_profile));\nreturn 0;}\n')
    exe = tmp_path / "lay"
    inc = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include")
    r = subprocess.run(["gcc", "-I", inc, str(src), "-o", str(exe)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    vals = [int(v) for v in subprocess.run([str(exe)], capture_output=True, text=True).stdout.split()]
    assert vals[0] == C.sizeof(cpqr.Options)
    assert vals[1:1 + len(fields)] == [getattr(cpqr.Options, f).offset for f in fields]
    assert vals[-1] == C.sizeof(cpqr.Profile)
