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
    hp = amgb.setup(p, c, v, reorder=0, **kw)
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


def test_reordered_level_ops_and_batched():
    """amg_level_op permutes each operand with its level's order; the row sums
    are formed exactly as on the plain store, so SpMV / residual / smoother /
    transfer results are bitwise equal; the batched solve matches per column."""
    p, c, v, f = synth.problem("poisson_perm", 30)
    hp = amgb.setup(p, c, v, reorder=0, coarse_enough=200)
    hr = amgb.setup(p, c, v, reorder=1, coarse_enough=200)
    for l in range(hp.nlevels - 1):
        n = hp.level_info(l)["rows"]
        nc = hp.level_info(l + 1)["rows"]
        x, fl, xc = synth.random_vector(n), synth.random_vector(n)[::-1].copy(), synth.random_vector(nc)
        for op, xin, fin, ny in ((amgb.OP_SPMV_A, x, None, n), (amgb.OP_RESIDUAL, x, fl, n),
                                 (amgb.OP_RELAX, x, fl, n), (amgb.OP_SPMV_P, xc, None, n),
                                 (amgb.OP_SPMV_R, x, None, nc)):
            ya = host(hp.level_op(l, op, x=dev(xin), f=dev(fin) if fin is not None else None, ny=ny))
            yb = host(hr.level_op(l, op, x=dev(xin), f=dev(fin) if fin is not None else None, ny=ny))
            assert np.array_equal(ya, yb), (l, op)
    F = torch.stack([dev(f), dev(f[::-1].copy()), dev(f * 0.5)])
    Xp, itp, _, stp = hp.solve_batched(F, tol=1e-8)
    Xr, itr, _, str_ = hr.solve_batched(F, tol=1e-8)
    assert stp == str_ == amgb.OK and np.max(np.abs(np.array(itp) - np.array(itr))) <= 1
    assert np.linalg.norm(host(Xr) - host(Xp)) <= 1e-7 * np.linalg.norm(host(Xp))


def test_automatic_reordering():
    """reorder = 2 (default): on for a randomly permuted matrix, off for a
    stencil in natural order (stats flags bit 1)."""
    for gen, expect in (("poisson_perm", 2), ("poisson", 0)):
        p, c, v, f = synth.problem(gen, 36)
        h = amgb.setup(p, c, v, coarse_enough=200)
        x, it, rel, st = h.solve(dev(f), tol=1e-8)
        assert st == amgb.OK and h.stats()["flags"] & 2 == expect, gen


def test_reordered_nonzero_initial_guess():
    p, c, v, f = synth.problem("poisson_perm", 20)
    hr = amgb.setup(p, c, v, reorder=1, coarse_enough=200)
    x0 = synth.random_vector(len(f))
    x, it, rel, st = hr.solve(dev(f), x=dev(x0), tol=1e-8)  # the initial guess is permuted too
    assert st == amgb.OK and rel <= 1.01e-8
