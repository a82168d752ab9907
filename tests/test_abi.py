"""The C ABI boundary: libwadg_b200.so loads without a GPU, exports every
entry point include/wadg_b200.h declares, and the ctypes mirror of
``wadg_problem`` has exactly the C layout (checked against gcc)."""

import ctypes
import os
import re
import subprocess

import pytest

from paper_1608_03836_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "wadg_b200.h")


def declared_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(wadg_[a-z0-9_]+)\s*\(", text)))


def test_library_loads_and_exports_every_declared_symbol():
    lib = _native.load()
    names = declared_functions()
    assert len(names) >= 10
    for name in names:
        assert hasattr(lib, name), name
        assert name in _native.EXPORTS, f"{name} has no ctypes prototype"
    assert lib.wadg_abi_version() == _native.ABI_VERSION


def test_struct_layout_matches_c(tmp_path):
    fields = [f[0] for f in _native.WadgProblem._fields_]
    src = ['#include <stdio.h>', '#include <stddef.h>', '#include "wadg_b200.h"', "int main(void) {",
           '  printf("size %zu\\n", sizeof(wadg_problem));']
    for f in fields:
        src.append(f'  printf("{f} %zu\\n", offsetof(wadg_problem, {f}));')
    src.append("  return 0; }")
    c = tmp_path / "layout.c"
    c.write_text("\n".join(src))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(c), "-o", str(exe)], check=True)
    out = dict(line.split() for line in subprocess.run([str(exe)], capture_output=True, text=True,
                                                        check=True).stdout.splitlines())
    assert int(out["size"]) == ctypes.sizeof(_native.WadgProblem)
    for f in fields:
        assert int(out[f]) == getattr(_native.WadgProblem, f).offset, f


def test_errors_are_reported_not_crashing():
    """Invalid arguments come back as nonzero codes with a message (no GPU
    work is launched for rejected problems)."""
    lib = _native.load()
    s = _native.WadgProblem()
    s.dim = 4
    rc = lib.wadg_volume(ctypes.byref(s), None, None, None)
    assert rc != 0 and b"dim" in lib.wadg_last_error()
    with pytest.raises(_native.NativeError):
        _native.call("wadg_volume", ctypes.byref(s), None, None, None)


def test_fused_configs_fit_shared_memory():
    for code in (_native.WADG_F32, _native.WADG_F64):
        for N in range(1, 8):
            cfg = _native.fused_config(code, N)
            assert cfg is not None, (code, N)
            assert cfg["smem"] <= 227 * 1024
