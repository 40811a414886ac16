"""The Python binding's ctypes mirrors of the C-ABI structs (include/amgb.h)
have the header's sizes and field offsets: a tiny C program compiled with gcc
against the header prints them.  CPU only (no library call)."""
import os
import shutil
import subprocess

import pytest

import paper_1811_05704_b200 as amgb

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PAIRS = [("amg_params", amgb.AmgParams), ("amg_level_info", amgb.LevelInfo),
         ("amg_level_export", amgb.LevelExport), ("amg_solve_stats", amgb.SolveStats),
         ("amg_dist", amgb.AmgDist), ("amg_dist_level_export", amgb.DistLevelExport),
         ("amg_level_op_args", amgb.LevelOpArgs)]


@pytest.mark.skipif(shutil.which("gcc") is None, reason="gcc not available")
def test_struct_layouts_match_header(tmp_path):
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "amgb.h"', "int main(void) {"]
    for cname, py in PAIRS:
        lines.append(f'  printf("{cname} size %zu\\n", sizeof({cname}));')
        for fname, _ in py._fields_:
            lines.append(f'  printf("{cname} {fname} %zu\\n", offsetof({cname}, {fname}));')
    lines += ["  return 0;", "}"]
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines) + "\n")
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-std=c11", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout.split("\n")
    got = {tuple(l.split()[:2]): int(l.split()[2]) for l in out if l.strip()}
    for cname, py in PAIRS:
        assert got[(cname, "size")] == __import__("ctypes").sizeof(py), cname
        for fname, _ in py._fields_:
            assert got[(cname, fname)] == getattr(py, fname).offset, (cname, fname)
