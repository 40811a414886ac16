"""Batched right-hand sides (amg_solve_batched): each column
must equal its own single-RHS solve (same iteration count, x to rounding) and
the oracle (iterations +-1, x within 1e-8).  GPU only."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
import paper_1811_05704_b200 as amgb  # noqa: E402
import synth  # noqa: E402


def rhs_block(n, k, seed=7):
    rng = np.random.default_rng(seed)
    F = rng.standard_normal((k, n))
    F[0] = 1.0  # the paper's f = 1
    return F


@pytest.mark.parametrize("k", [1, 3, 4, 8])
@pytest.mark.parametrize("gen,n,kw", [("poisson", 24, {}), ("varcoef", 18, {"relax": "chebyshev"}),
                                      ("poisson_perm", 16, {"npre": 2, "npost": 2})])
def test_batched_matches_single_and_oracle(k, gen, n, kw):
    p, c, v, f = synth.problem(gen, n)
    kw = dict(kw, coarse_enough=100)
    h = amgb.setup(p, c, v, **kw)
    F = rhs_block(len(f), k)
    Fd = torch.from_numpy(F).cuda()
    X, its, rels, st = h.solve_batched(Fd, tol=1e-8, maxiter=100)
    assert st == amgb.OK
    Xh = X.cpu().numpy()
    A = oracle.Csr(p, c, v)
    hier = oracle.Hierarchy(A, **kw)
    for j in range(k):
        xs, it_s, rel_s, st_s = h.solve(Fd[j].clone(), tol=1e-8, maxiter=100)
        assert its[j] == it_s, (j, its[j], it_s)
        assert np.linalg.norm(Xh[j] - xs.cpu().numpy()) <= 1e-10 * np.linalg.norm(Xh[j])
        assert rels[j] <= 1.01e-8
        o = oracle.cg(A, F[j], tol=1e-8, maxiter=100, hier=hier)
        assert abs(its[j] - o["iters"]) <= 1
        if its[j] == o["iters"]:
            assert np.linalg.norm(Xh[j] - o["x"]) <= 1e-8 * np.linalg.norm(o["x"])


def test_batched_zero_column_initial_guess_and_maxiter():
    p, c, v, f = synth.problem("poisson", 20)
    h = amgb.setup(p, c, v, coarse_enough=100)
    n = len(f)
    F = rhs_block(n, 3)
    F[1] = 0.0
    X0 = np.ones((3, n))
    X, its, rels, st = h.solve_batched(torch.from_numpy(F).cuda(), torch.from_numpy(X0).cuda(), tol=1e-8)
    Xh = X.cpu().numpy()
    assert its[1] == 0 and np.all(Xh[1] == 0) and rels[1] == 0
    for j in (0, 2):  # from a non-zero initial guess, vs the single solve from the same guess
        xs, it_s, _, _ = h.solve(torch.from_numpy(F[j]).cuda(), torch.from_numpy(X0[j]).cuda(), tol=1e-8)
        assert its[j] == it_s and np.linalg.norm(Xh[j] - xs.cpu().numpy()) <= 1e-10 * np.linalg.norm(Xh[j])
    X, its, rels, st = h.solve_batched(torch.from_numpy(F).cuda(), tol=0.0, maxiter=3)
    assert st == amgb.NOT_CONVERGED and list(its) == [3, 0, 3]


def test_batched_errors():
    p, c, v, f = synth.problem("poisson", 12)
    h = amgb.setup(p, c, v, coarse_enough=100)
    with pytest.raises(amgb.AmgError):
        h.solve_batched(torch.zeros((9, len(f)), dtype=torch.float64, device="cuda"))
    hb = amgb.setup(p, c, v, coarse_enough=100, solver="bicgstab")
    with pytest.raises(amgb.AmgError):
        hb.solve_batched(torch.zeros((2, len(f)), dtype=torch.float64, device="cuda"))
