"""T2: the library's host setup (libamgb.so, host-only handle) against the
oracle: aggregates and sparsity patterns bit-exact, values within 1e-12
relative (in practice bit-exact: both sum in ascending index order without FP
contraction, DESIGN.md §3 R7/R28).  CPU only, through the C ABI."""
import numpy as np
import pytest

import oracle
import paper_1811_05704_b200 as amgb
import synth

CASES = [
    ("poisson", 24, {}),
    ("poisson", 32, {}),
    ("poisson_perm", 20, {}),
    ("varcoef", 20, {"relax": "chebyshev"}),
    ("varcoef", 22, {}),
    ("convdiff", 18, {"relax": "damped_jacobi"}),
    ("poisson", 20, {"coarsening": 1}),
    ("poisson", 20, {"coarse_enough": 50, "npre": 2}),
]

ORACLE_KW = {"coarsening": "smoothed"}


def _okw(kw):
    o = dict(kw)
    if "coarsening" in o:
        o["smoothed"] = 1 - o.pop("coarsening")
    o.pop("npre", None)
    return o


def _same_csr(a, b, rel=1e-12):
    ptr, col, val = a
    assert np.array_equal(ptr, b.ptr)
    assert np.array_equal(col, b.col)
    scale = max(np.abs(b.val).max(initial=0.0), 1e-300)
    assert np.max(np.abs(val - b.val), initial=0.0) <= rel * scale


@pytest.mark.parametrize("gen,n,kw", CASES)
def test_host_setup_matches_oracle(gen, n, kw):
    p, c, v, f = synth.problem(gen, n)
    h = amgb.setup(p, c, v, device=-1, **kw)
    o = oracle.Hierarchy(oracle.Csr(p, c, v), **_okw(kw))
    assert h.nlevels == o.nlevels
    for l in range(h.nlevels):
        e = h.export_level(l)
        _same_csr(e["A"], o.matrix(l, "A"))
        if l < h.nlevels - 1:
            assert np.array_equal(e["aggregates"], o.aggregates(l))
            _same_csr(e["P"], o.matrix(l, "P"))
            _same_csr(e["R"], o.matrix(l, "R"))
            np.testing.assert_allclose(e["smoother"], o.smoother(l), rtol=1e-14, atol=0)
        else:
            inv = e["coarse_inverse"]
            A = o.matrix(l, "A").to_dense()
            assert np.abs(inv @ A - np.eye(len(A))).max() <= 1e-10


def test_info_counts():
    p, c, v, f = synth.poisson3d(16)
    h = amgb.setup(p, c, v, device=-1, coarse_enough=100)
    inf = [h.level_info(l) for l in range(h.nlevels)]
    assert inf[0]["rows"] == 4096 and inf[0]["nnz_A"] == len(c)
    for a, b in zip(inf, inf[1:]):
        assert a["cols_P"] == b["rows"] and a["aggregates"] == a["cols_P"]
    assert inf[-1]["is_coarsest"] == 1 and inf[-1]["nnz_P"] == 0
    assert all(i["alg_bytes_vcycle"] > 0 for i in inf)


def test_setup_errors():
    # bad CSR: unsorted columns
    with pytest.raises(amgb.AmgError) as e:
        amgb.setup(np.array([0, 2, 3]), np.array([1, 0, 1]), np.ones(3), device=-1, coarse_enough=1)
    assert e.value.code == amgb.E_BAD_CSR
    # non-positive diagonal
    with pytest.raises(amgb.AmgError) as e:
        amgb.setup(np.array([0, 2, 4]), np.array([0, 1, 0, 1]), np.array([-1.0, 1, 1, 2]),
                   device=-1, coarse_enough=1)
    assert e.value.code == amgb.E_ZERO_DIAG
    # singular coarse
    with pytest.raises(amgb.AmgError) as e:
        amgb.setup(np.array([0, 2, 4]), np.array([0, 1, 0, 1]), np.array([1.0, 1, 1, 1]),
                   device=-1)
    assert e.value.code == amgb.E_SINGULAR_COARSE
    # too large coarsest
    p, c, v, f = synth.poisson3d(6)
    with pytest.raises(amgb.AmgError) as e:
        amgb.setup(p, c, v, device=-1, dense_max=10)
    assert e.value.code == amgb.E_COARSE_TOO_LARGE
    # bad params
    with pytest.raises(amgb.AmgError) as e:
        amgb.setup(p, c, v, device=-1, relax=7)
    assert e.value.code == amgb.E_INVALID_ARG
    with pytest.raises(KeyError):
        amgb.make_params({"no.such.key": 1})
    # solve on a host-only handle
    h = amgb.setup(p, c, v, device=-1)
    with pytest.raises(amgb.AmgError) as e:
        h.solve_host(f)
    assert e.value.code == amgb.E_NO_DEVICE


def test_dotted_param_keys():
    prm = amgb.make_params({"solver.type": "bicgstab", "precond.relax.type": "chebyshev",
                            "precond.coarsening.type": "aggregation"})
    assert prm.solver == 1 and prm.relax == 2 and prm.coarsening == 1


def test_vector_length_and_host_checks():
    """amg_vector_length on a host-only handle (the global n) and the binding's
    host-array checks (no GPU needed: they run before any library call)."""
    p, c, v, f = synth.poisson3d(10, 11, 12)
    h = amgb.setup(p, c, v, device=-1)
    assert h.vec_len == len(f) == 10 * 11 * 12
    with pytest.raises(ValueError):
        amgb._host_vec(np.zeros(5), 6, "f")
    with pytest.raises(ValueError):
        amgb._host_vec(np.zeros(6, np.float32), 6, "f")
    with pytest.raises(ValueError):
        amgb._host_vec(np.zeros((6, 2))[:, 0], 6, "f")
    assert amgb._host_vec(np.zeros(6), 6, "f").shape == (6,)
