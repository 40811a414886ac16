"""Locality reordering of the device store (params reorder = 1):
the same hierarchy stored in reverse-Cuthill-McKee order (aggregates numbered
by their roots), vectors permuted at the API.  Every row sum is formed from the
same entries in the same order; only the dense coarse GEMV and the Krylov dots
sum in another order, so results agree to rounding.  GPU only."""
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


@pytest.mark.parametrize("gen,n,kw", [("poisson_perm", 40, {}), ("poisson", 33, {}),
                                      ("varcoef", 24, {"relax": "chebyshev"}),
                                      ("convdiff", 20, {"relax": "damped_jacobi", "solver": "bicgstab"}),
                                      ("convdiff", 20, {"solver": "idrs"}), ("convdiff", 18, {"solver": "gmres"})])
def test_reordered_store_matches(gen, n, kw):
    p, c, v, f = synth.problem(gen, n)
    kw = dict(kw, coarse_enough=200)
    hp = amgb.setup(p, c, v, **kw)
    hr = amgb.setup(p, c, v, reorder=1, **kw)
    r = synth.random_vector(len(f))
    zp, zr = host(hp.precond(dev(r))), host(hr.precond(dev(r)))
    assert np.linalg.norm(zr - zp) <= 1e-12 * np.linalg.norm(zp)
    xp, itp, relp, stp = hp.solve(dev(f), tol=1e-8, maxiter=300)
    xr, itr, relr, str_ = hr.solve(dev(f), tol=1e-8, maxiter=300)
    assert stp == str_ == amgb.OK and abs(itp - itr) <= 1 and relr <= 1.01e-8
    A = oracle.Csr(p, c, v)
    res = f - oracle.spmv(A, host(xr))
    assert np.linalg.norm(res) <= 1.01e-8 * np.linalg.norm(f)
    if itp == itr:
        assert np.linalg.norm(host(xr) - host(xp)) <= 1e-7 * np.linalg.norm(host(xp))
    xh, ith, relh, sth = hr.solve_host(f, tol=1e-8, maxiter=300)
    assert ith == itr and np.array_equal(xh, host(xr))


def test_reordered_store_limits():
    p, c, v, f = synth.problem("poisson_perm", 20)
    hr = amgb.setup(p, c, v, reorder=1, coarse_enough=200)
    with pytest.raises(amgb.AmgError):
        hr.level_op(0, amgb.OP_SPMV_A, x=dev(f), ny=len(f))
    with pytest.raises(amgb.AmgError):
        hr.solve_batched(torch.stack([dev(f)] * 2))
    x0 = synth.random_vector(len(f))
    x, it, rel, st = hr.solve(dev(f), x=dev(x0), tol=1e-8)  # non-zero initial guess is permuted too
    assert st == amgb.OK and rel <= 1.01e-8
