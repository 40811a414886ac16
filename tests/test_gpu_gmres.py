"""Restarted right-preconditioned GMRES(m) on the GPU (solver = 2) against the
oracle's GMRES(m) (modified Gram-Schmidt; the GPU uses classical Gram-Schmidt
applied twice -- same algorithm up to rounding): iterations within +-1, and at
equal iteration count |x - x_oracle| <= 1e-8 |x_oracle|.  GPU only."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
import paper_1811_05704_b200 as amgb  # noqa: E402
import synth  # noqa: E402


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, np.float64)).cuda()


@pytest.mark.parametrize("gen,n,kw,m", [
    ("convdiff", 24, {"relax": "damped_jacobi"}, 30),
    ("convdiff", 20, {"relax": "damped_jacobi"}, 4),     # several restart cycles
    ("poisson", 28, {}, 30),
    ("varcoef", 20, {"relax": "chebyshev"}, 8),
])
def test_gmres_matches_oracle(gen, n, kw, m):
    p, c, v, f = synth.problem(gen, n)
    kw = dict(kw, coarse_enough=100)
    h = amgb.setup(p, c, v, {"solver.type": "gmres", "solver.M": m}, **kw)
    A = oracle.Csr(p, c, v)
    hier = oracle.Hierarchy(A, **kw)
    o = oracle.gmres(A, f, tol=1e-8, maxiter=300, m=m, hier=hier)
    x, it, rel, st = h.solve(dev(f), tol=1e-8, maxiter=300)
    assert st == amgb.OK and o["status"] == oracle.OK
    assert abs(it - o["iters"]) <= 1, (it, o["iters"])
    assert rel <= 1e-8
    true = np.linalg.norm(f - oracle.spmv(A, x.cpu().numpy())) / np.linalg.norm(f)
    assert abs(true - rel) <= 1e-12
    if it != o["iters"]:
        x, it, rel, st = h.solve(dev(f), tol=0.0, maxiter=o["iters"])
    assert np.linalg.norm(x.cpu().numpy() - o["x"]) <= 1e-8 * np.linalg.norm(o["x"])
    s = h.stats()
    assert s["vcycles"] >= s["iters"] + 1


def test_gmres_zero_rhs_maxiter_and_params():
    p, c, v, f = synth.problem("convdiff", 12)
    h = amgb.setup(p, c, v, {"solver.type": "gmres", "solver.M": 5}, coarse_enough=100, relax="damped_jacobi")
    x, it, rel, st = h.solve(dev(np.zeros_like(f)), x=dev(np.ones_like(f)))
    assert it == 0 and st == amgb.OK and np.all(x.cpu().numpy() == 0)
    x, it, rel, st = h.solve(dev(f), tol=0.0, maxiter=7)
    o = oracle.gmres(oracle.Csr(p, c, v), f, tol=0.0, maxiter=7, m=5,
                     hier=oracle.Hierarchy(oracle.Csr(p, c, v), coarse_enough=100, relax="damped_jacobi"))
    assert it == 7 == o["iters"] and st == amgb.NOT_CONVERGED
    assert np.linalg.norm(x.cpu().numpy() - o["x"]) <= 1e-9 * np.linalg.norm(o["x"])
    with pytest.raises(amgb.AmgError):
        amgb.setup(p, c, v, {"solver.type": "gmres", "solver.M": 0}, device=-1)
