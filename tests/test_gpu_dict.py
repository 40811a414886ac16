"""Column-offset dictionary of the TMA-staged SELL-32 format:
slices whose 32 rows share one offset list store it once.  It is a storage
choice only: the row sums are formed from the same entries in the same column
order (a row missing an offset contributes 0 * x_j), so every result must be
BITWISE equal to the explicit-index format (AMGB_NO_DICT=1) and within the
usual tolerance of the oracle.  GPU only."""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
import paper_1811_05704_b200 as amgb  # noqa: E402
import synth  # noqa: E402


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, np.float64)).cuda()


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


def setup_both(p, c, v, **kw):
    h_dict = amgb.setup(p, c, v, **kw)
    os.environ["AMGB_NO_DICT"] = "1"
    try:
        h_plain = amgb.setup(p, c, v, **kw)
    finally:
        del os.environ["AMGB_NO_DICT"]
    return h_dict, h_plain


# 48^3 / 41^3: level-0 A has >= 65536 rows of <= 7 entries -> TMA format; the
# boundary planes exercise rows missing offsets and the first/last z-planes
# (row + offset out of range) stay explicit.  41^3: a ragged last slice.
@pytest.mark.parametrize("n", [48, 41])
def test_dictionary_bitwise_equal(n):
    p, c, v, f = synth.problem("poisson", n)
    hd, hp = setup_both(p, c, v)
    info = hd.level_info(0)
    nslices = (len(f) + 31) // 32
    assert info["dict_slices_A"] > nslices // 2, info
    assert hp.level_info(0)["dict_slices_A"] == 0
    A = oracle.Csr(p, c, v)
    xin = synth.random_vector(len(f))
    yd = host(hd.level_op(0, amgb.OP_SPMV_A, x=dev(xin), ny=len(f)))
    yp = host(hp.level_op(0, amgb.OP_SPMV_A, x=dev(xin), ny=len(f)))
    assert np.array_equal(yd, yp)
    ref = oracle.spmv(A, xin)
    assert np.max(np.abs(yd - ref)) <= 1e-12 * np.max(np.abs(ref))
    xd, itd, reld, _ = hd.solve(dev(f), tol=1e-8)
    xp, itp, relp, _ = hp.solve(dev(f), tol=1e-8)
    assert itd == itp and reld == relp
    assert np.array_equal(host(xd), host(xp))
    o = oracle.cg(A, f, tol=1e-8, maxiter=100, hier=oracle.Hierarchy(A))
    assert abs(itd - o["iters"]) <= 1
    if itd == o["iters"]:
        assert np.linalg.norm(host(xd) - o["x"]) <= 1e-8 * np.linalg.norm(o["x"])


def test_dictionary_mixed_precision_and_varcoef():
    p, c, v, f = synth.problem("varcoef", 42)
    hd, hp = setup_both(p, c, v, precision="mixed", relax="chebyshev")
    assert hd.level_info(0)["dict_slices_A"] > 0
    r = synth.random_vector(len(f))
    assert np.array_equal(host(hd.precond(dev(r))), host(hp.precond(dev(r))))
    xd, itd, _, _ = hd.solve(dev(f), tol=1e-8)
    xp, itp, _, _ = hp.solve(dev(f), tol=1e-8)
    assert itd == itp and np.array_equal(host(xd), host(xp))


def test_no_dictionary_for_unstructured_rows():
    p, c, v, f = synth.problem("poisson_perm", 48)
    h = amgb.setup(p, c, v)
    assert h.level_info(0)["dict_slices_A"] == 0
