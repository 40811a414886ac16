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


def test_params_defaults_and_validation_host_only():
    """New parameters: defaults (GPU setup on, IDR(s) s = 4) and their validation,
    checked on host-only handles (device = -1, no GPU needed)."""
    import numpy as np
    import pytest

    import synth
    p = amgb.make_params()
    assert p.setup_device == 1 and p.idrs_s == 4 and p.solver == 0
    assert amgb.make_params(solver="idrs", **{"solver.s": 8}).idrs_s == 8
    ptr, col, val, f = synth.problem("poisson", 10)
    h = amgb.setup(ptr, col, val, device=-1, setup_device="gpu", coarse_enough=100)  # host build
    assert h.nlevels >= 2
    for bad in ({"solver": "idrs", "idrs_s": 3}, {"setup_device": 2}, {"solver": 4}):
        with pytest.raises(amgb.AmgError) as e:
            amgb.setup(ptr, col, val, device=-1, **bad)
        assert e.value.code == amgb.E_INVALID_ARG
    assert np.isfinite(h.level_info(0)["alg_bytes_vcycle"])


def test_host_only_handle_rejects_solves_and_reports_store_fields():
    """amg_solve_host_stream needs a device handle (error, not a crash, on a
    host-only handle); level info of a host-only handle has no device store."""
    import numpy as np
    import pytest

    import synth
    ptr, col, val, f = synth.problem("poisson", 10)
    h = amgb.setup(ptr, col, val, device=-1, coarse_enough=100)
    with pytest.raises(amgb.AmgError) as e:
        h.solve_host_stream([f, f])
    assert e.value.code < 0 and "amg_solve_host_stream failed" in str(e.value)
    info = h.level_info(0)
    assert info["padded_nnz_P"] == 0 and info["padded_nnz_R"] == 0 and info["sigma_mask"] == 0
    assert info["nnz_P"] > 0 and np.isfinite(info["alg_bytes_vcycle"])
