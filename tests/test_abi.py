"""The C-ABI library loads without a GPU and exports every symbol that
include/amgb.h declares; no compute calls."""
import ctypes
import os
import re
import subprocess

import paper_1811_05704_b200 as amgb

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "amgb.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(amg_[a-z_]+)\s*\(", src)))


def test_header_symbols_exported():
    names = declared_functions()
    assert len(names) >= 14
    lib = ctypes.CDLL(amgb.LIB_PATH)
    for n in names:
        assert hasattr(lib, n), n
    out = subprocess.run(["nm", "-D", "--defined-only", amgb.LIB_PATH], capture_output=True,
                         text=True).stdout
    for n in names:
        assert re.search(rf"\bT {n}$", out, re.M), n
    assert set(amgb.SYMBOLS) == set(names)


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", amgb.LIB_PATH], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_params_struct_size():
    p = amgb.make_params()
    assert p.struct_size == ctypes.sizeof(amgb.AmgParams)
    assert abs(p.p_omega - 2 / 3) < 1e-16 and p.eps_strong == 0.08 and p.coarse_enough == 3000
    assert "sm_100a" in amgb.version()
