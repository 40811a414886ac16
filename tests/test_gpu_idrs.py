"""IDR(s) on the device (solver = "idrs"; idrs.cuh) against
the oracle's or_idrs (pinned in tests/test_oracle_idrs.py).  The device takes the
bi-orthogonalisation coefficients from one set of dots P^T (A U_k) instead of
the oracle's one-at-a-time projections (same numbers in exact arithmetic), and
its reductions sum in a different order, so the bar is rounding-level: after a
fixed number of products (tol = 0) x agrees to 1e-9 relative; converged solves
agree in iteration count within +-2 and in x within 1e-6 (both satisfy
|f - A x| <= 1e-8 |f|).  The shadow space is the same counter-based generator
on both sides.  GPU only."""
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


@pytest.mark.parametrize("s", [1, 2, 4, 8])
def test_idrs_fixed_steps_match_oracle(s):
    p, c, v, f = synth.problem("convdiff", 16)
    kw = dict(coarse_enough=100, relax="damped_jacobi")
    h = amgb.setup(p, c, v, solver="idrs", idrs_s=s, **kw)
    A = oracle.Csr(p, c, v)
    H = oracle.Hierarchy(A, **kw)
    for k in sorted({1, 2, s, s + 1, s + 2, 2 * (s + 1) + 1}):
        x, it, rel, st = h.solve(dev(f), tol=0.0, maxiter=k)
        o = oracle.idrs(A, f, tol=0.0, maxiter=k, s=s, hier=H)
        assert it == o["iters"] == k
        xo = o["x"]
        assert np.linalg.norm(host(x) - xo) <= 1e-9 * np.linalg.norm(xo), (s, k)
        assert h.stats()["vcycles"] == k


CASES = [("convdiff", 20, 4, {"relax": "damped_jacobi"}), ("convdiff", 20, 2, {}),
         ("poisson", 32, 4, {}), ("varcoef", 20, 4, {"relax": "chebyshev"}), ("poisson_perm", 20, 8, {})]


@pytest.mark.parametrize("gen,n,s,kw", CASES)
def test_idrs_converged_solve_matches_oracle(gen, n, s, kw):
    p, c, v, f = synth.problem(gen, n)
    kw = dict(kw, coarse_enough=100)
    h = amgb.setup(p, c, v, solver="idrs", idrs_s=s, **kw)
    x, it, rel, st = h.solve(dev(f), tol=1e-8, maxiter=300)
    assert st == amgb.OK and rel <= 1e-8
    A = oracle.Csr(p, c, v)
    o = oracle.idrs(A, f, tol=1e-8, maxiter=300, s=s, hier=oracle.Hierarchy(A, **kw))
    assert o["status"] == 0
    # north-star bar: iterations (preconditioned products) +-1, x within 1e-8 at
    # equal count (a run that stops one product apart is re-run at the oracle's)
    assert abs(it - o["iters"]) <= 1, (it, o["iters"])
    xh = host(x)
    r = f - oracle.spmv(A, xh)
    assert np.linalg.norm(r) <= 1.01e-8 * np.linalg.norm(f)
    if it != o["iters"]:
        x, it, rel, st = h.solve(dev(f), tol=0.0, maxiter=o["iters"])
        assert it == o["iters"]
        xh = host(x)
    assert np.linalg.norm(xh - o["x"]) <= 1e-8 * np.linalg.norm(o["x"])


def test_idrs_edge_cases():
    p, c, v, f = synth.problem("convdiff", 12)
    h = amgb.setup(p, c, v, solver="idrs", coarse_enough=100)
    x, it, rel, st = h.solve(dev(np.zeros_like(f)), x=dev(np.ones_like(f)))
    assert it == 0 and st == amgb.OK and np.all(host(x) == 0)
    x, it, rel, st = h.solve(dev(f), tol=1e-8, maxiter=0)
    assert it == 0 and st == amgb.NOT_CONVERGED
    xh, it2, rel2, st2 = h.solve_host(f, tol=1e-8)
    xd, it3, rel3, st3 = h.solve(dev(f), tol=1e-8)
    assert it2 == it3 and st2 == st3 == amgb.OK
    assert np.array_equal(xh, host(xd))
    # graph replay == direct launches
    hn = amgb.setup(p, c, v, solver="idrs", coarse_enough=100, use_graph=0)
    xn, it4, _, _ = hn.solve(dev(f), tol=1e-8)
    assert it4 == it3 and np.array_equal(host(xn), host(xd))
    with pytest.raises(amgb.AmgError):
        amgb.setup(p, c, v, solver="idrs", idrs_s=3)
