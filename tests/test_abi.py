"""The C ABI library loads and exports every symbol include/sgb.h declares."""

import ctypes
import re
from pathlib import Path

import numpy as np

from paper_2110_12865_b200 import runtime
from paper_2110_12865_b200.lower import GROUP_DTYPE

HDR = Path(__file__).resolve().parent.parent / "include" / "sgb.h"


def declared_functions():
    text = HDR.read_text()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|void|const char \*)\s*\*?\s*(sgb_\w+)\s*\(", text, re.M)))


def test_header_declares_the_runtime_symbols():
    assert set(declared_functions()) == set(runtime.SYMBOLS)


def test_library_exports_every_declared_symbol():
    lib = runtime.load_library()
    for name in declared_functions():
        assert hasattr(lib, name), name


def test_group_record_matches_header():
    # sgb_group: 11 int64 + 14 int32 (the gcc probe below checks every offset)
    assert GROUP_DTYPE.itemsize == 11 * 8 + 14 * 4


def test_desc_layout_matches_header(tmp_path):
    """Compile the header with gcc and compare every field offset with ctypes."""
    import shutil
    import subprocess

    import pytest

    if not shutil.which("gcc"):
        pytest.skip("no gcc")
    fields = [f for f, _ in runtime._Desc._fields_]
    gfields = list(GROUP_DTYPE.names)
    src = tmp_path / "probe.c"
    src.write_text(
        '#include <stdio.h>\n#include <stddef.h>\n#include "sgb.h"\nint main(void){\n'
        + 'printf("%zu\\n", sizeof(sgb_plan_desc));\n'
        + "".join(f'printf("%zu\\n", offsetof(sgb_plan_desc, {f}));\n' for f in fields)
        + 'printf("%zu\\n", sizeof(sgb_group));\n'
        + "".join(f'printf("%zu\\n", offsetof(sgb_group, {f}));\n' for f in gfields)
        + "return 0;}\n")
    exe = tmp_path / "probe"
    subprocess.run(["gcc", "-I", str(HDR.parent), "-o", str(exe), str(src)], check=True)
    got = [int(v) for v in subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()]
    want = [ctypes.sizeof(runtime._Desc)] + [getattr(runtime._Desc, f).offset for f in fields]
    want += [GROUP_DTYPE.itemsize] + [GROUP_DTYPE.fields[f][1] for f in gfields]
    assert got == want


def test_last_error_is_a_string():
    lib = runtime.load_library()
    assert isinstance(lib.sgb_last_error(), bytes)


def test_create_rejects_null_descriptor():
    lib = runtime.load_library()
    out = ctypes.c_void_p(0)
    rc = lib.sgb_plan_create(None, 0, ctypes.byref(out))
    assert rc != 0 and not out.value
    assert lib.sgb_last_error()
